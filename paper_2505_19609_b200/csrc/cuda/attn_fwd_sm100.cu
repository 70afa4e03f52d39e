// Row a7: packed varlen causal attention forward on sm_100a (tcgen05 + TMEM + TMA).
//
// Work unit (CTA): one 128-row query tile of one segment x two q-heads of the same KV group
// (GQA, R30), so each K/V tile is loaded once into shared memory and feeds both heads (d = 128 with
// an odd group: one pair in each straddles two groups and streams both groups' K/V, see the kernel).
// Warp roles (576 threads):
//   warps 0-7  softmax of head A (ha): two warpgroups split the 128 key columns of each S tile
//              (warpgroup 0 keys [0,64), warpgroup 1 keys [64,128)); thread = query row of the tile,
//              the two halves of a row combine their maxima through shared memory once per tile
//   warps 8-15 softmax of head B (hb = ha + 1, if it exists), same split
//   warp 16    TMA producer: Q tiles once, then a ring of K/V tiles (SW128, 64-col boxes)
//   warp 17    MMA issuer (one thread): S = Q K^T into TMEM, O += P V into TMEM; S(j+1) is issued as
//              soon as the softmax has read S(j) (s_free), overlapping the exponentials of tile j
// Two warpgroups per head halve the per-head softmax chain (S(j) -> exps -> P(j) -> PV(j) -> S(j+1)
// is serial per head when P aliases S) and put four softmax warps on every sub-partition.
// TMEM (512 cols): see Cfg.
// Softmax: S row read with tcgen05.ld (no shuffles: one thread = one row), exp2 with the scale
// folded in, running max kept in log2 units and O rescaled in TMEM only when the max grows by
// more than 8 (exact: the final normalisation uses the same reference max), P written as bf16 pairs
// into TMEM with tcgen05.st and fed to the PV MMA as its A operand straight from TMEM (no smem
// traffic: with single-CTA M=128 MMAs the SS operand reads alone saturate shared memory). Causal: only KV tiles up to the tile's last
// query are visited (bottom-right aligned with q_pos, R23); the diagonal tiles are masked.
#include <cstdlib>

#include "attn_common.cuh"
#include "device.cuh"
#include "sm100.cuh"
#include "tma.h"

namespace skr {
namespace fwd {

// Debug timeline (SKR_TRACE=1): (event, clock) pairs of block (0, 0) into a device buffer.
__device__ unsigned long long* g_trace = nullptr;
// fire-and-forget store (no atomics: a returning atomic would cost ~1000 cycles on the traced path);
// each recording thread owns a 2048-entry slice chosen by its role
__shared__ int g_trace_cnt[8];
__shared__ unsigned long long* g_trace_smem;   // this block's buffer (null: not traced), read from smem
__device__ __forceinline__ void trace_init() {
#if defined(SKR_KERNEL_TRACE) || defined(SKR_PHASE_ACCT)
  if (threadIdx.x < 8) g_trace_cnt[threadIdx.x] = 0;
  if (threadIdx.x == 0) g_trace_smem = (blockIdx.x == 0 && blockIdx.y == 0) ? g_trace : nullptr;
#endif
}
__device__ __forceinline__ void trace(int ev, int j = 0) {   // j: tile index payload (8 bits)
#ifdef SKR_KERNEL_TRACE   // debug builds only: production kernels carry no instrumentation
  unsigned long long* buf = g_trace_smem;
  if (buf != nullptr) {
    const int role = ev / 10 < 8 ? ev / 10 : 7;
    const int i = g_trace_cnt[role]++;
    buf[role * 1024 + (i & 1023)] = ((unsigned long long)ev << 48) | ((unsigned long long)(j & 0xFF) << 40) |
                                     (clock64() & 0xFFFFFFFFFFull);
  }
#endif
}
// per-warp event (several warps share the role slice: shared atomic slot), debug builds only
__device__ __forceinline__ void trace_w(int ev, int j) {
#ifdef SKR_KERNEL_TRACE
  unsigned long long* buf = g_trace_smem;
  if (buf != nullptr) {
    const int role = ev / 10 < 8 ? ev / 10 : 7;
    const int i = atomicAdd(&g_trace_cnt[role], 1);
    buf[role * 1024 + (i & 1023)] = ((unsigned long long)ev << 48) | ((unsigned long long)(j & 0xFF) << 40) |
                                     (clock64() & 0xFFFFFFFFFFull);
  }
#endif
}

// softmax-side events perturb the warpgroup they are recorded from (the traced warp falls behind
// its siblings and every 128-arrival barrier waits for it): separate opt-in, SKR_TRACE_SOFTMAX
#ifdef SKR_TRACE_SOFTMAX
__device__ __forceinline__ void trace_sm(int ev, int j) { trace(ev, j); }
__device__ __forceinline__ void trace_smw(int ev, int j) { trace_w(ev, j); }
#else
__device__ __forceinline__ void trace_sm(int, int) {}
__device__ __forceinline__ void trace_smw(int, int) {}
#endif

constexpr int BM = 128, BN = 128;

// A tile whose queries see no key at all (ring CP: a key chunk after the query chunk, k_len = 0):
// O = 0 and LSE = -inf, the neutral element of the partial-attention merge. Written by the whole CTA
// before any barrier / TMEM is set up; the caller returns right after (the condition is CTA-uniform).
template <int D>
__device__ __forceinline__ void store_empty_tile(const AttnArgs& a, __nv_bfloat16* __restrict__ out,
                                                 float* __restrict__ lse, int r0, int n_valid, int h0, int nh) {
  const int per_row = nh * (D / 8);                     // 16-byte vectors per query row
  for (int e = threadIdx.x; e < n_valid * per_row; e += blockDim.x) {
    const int row = e / per_row, rem = e % per_row, hh = rem / (D / 8), c = rem % (D / 8);
    *reinterpret_cast<uint4*>(out + ((size_t)(r0 + row) * a.hq + h0 + hh) * D + c * 8) = make_uint4(0u, 0u, 0u, 0u);
  }
  for (int e = threadIdx.x; e < n_valid * nh; e += blockDim.x)
    lse[(size_t)(h0 + e / n_valid) * a.ld_lse + r0 + e % n_valid] = -INFINITY;
}
constexpr int kThreads = 576;
// Grid order of the two-head kernel (launch argument head_major): 0 = (head pair, tile) with the
// pair fastest; 1 = (tile, head pair), every tile of one pair before the next pair, so the CTAs in
// flight share one KV head's K / V (L2-resident) instead of streaming every head's. d = 128 uses 1:
// S4n1 fwd DRAM 52 -> 9.4 GB per launch, S4n1 / C5n1 +2 % / +6 % (profiles/r02_experiments.md);
// d = 64 keeps 0 (a 32K sequence's K / V is 8 MB per head, L2-resident either way; 1 measured -1.5 %).
constexpr int kSoftmax = 256;                // threads per head (two warpgroups)
constexpr int kTmaWarp = 16, kMmaWarp = 17;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

// softmax warpgroups per head of the d = 128 two-head forward (see attn_fwd_kernel's kWG)
#ifndef SKR_FWD_WG128
#define SKR_FWD_WG128 2
#endif
#ifndef SKR_FWD_WG64
#define SKR_FWD_WG64 2
#endif

#ifndef SKR_FWD_BN128
#define SKR_FWD_BN128 128   // key-tile width of the d = 128 forward (64: separate P columns, see Cfg)
#endif

#ifndef SKR_FWD_ROWSPLIT
#define SKR_FWD_ROWSPLIT 1
#endif
// SKR_FWD_SSPLIT (experiment, d = 128 row split): P goes to the SECOND half of S's columns and
// S(j+1) is issued as two N = 64 halves -- the first (keys [0, 64), columns [0, 64)) as soon as the
// softmax has loaded S(j), the second after PV(j) -- so only PV + half an S stay on each head's chain.
#ifndef SKR_FWD_SSPLIT
#define SKR_FWD_SSPLIT 0
#endif
#ifndef SKR_FWD_ORDER64
#define SKR_FWD_ORDER64 0
#endif
#ifndef SKR_FWD_PVFIRST
#define SKR_FWD_PVFIRST 1   // MMA thread: PV_A(j-1) before the K(j) wait (S4n1 fwd -2 %, r02_run31)
#endif

template <int D>
struct Cfg {
  static constexpr int BN = D == 128 ? SKR_FWD_BN128 : 128;   // keys per K/V tile
  static constexpr int kChunks = D / 64;                 // 64-col SW128 boxes per row
  static constexpr int kQBytes = BM * D * 2;             // one Q tile
  static constexpr int kKVBytes = BN * D * 2;            // one K or V tile
#ifndef SKR_FWD_UNITS64
#define SKR_FWD_UNITS64 6
#endif
#ifndef SKR_FWD_UNITS128
#define SKR_FWD_UNITS128 4
#endif
  static constexpr int kUnits = D == 128 ? (BN == 64 ? 8 : SKR_FWD_UNITS128) : SKR_FWD_UNITS64;   // K/V ring depth (tiles), <= 8
  static constexpr int kOffQ = 0;
  static constexpr int kOffKV = 2 * kQBytes;
  static constexpr int kOffRed = kOffKV + kUnits * kKVBytes;   // [head][tile parity][half][row] row maxima
  // (the row-split softmax exchanges nothing through shared memory: no reduction buffer)
  static constexpr int kOffBar = kOffRed + (SKR_FWD_ROWSPLIT ? 0 : 2 * 2 * 2 * BM * 4);
  static constexpr int kSmem = kOffBar + 256 + 1024;    // + barriers + alignment slack
  // TMEM columns. P (bf16 pairs) is the A operand of O += P V straight from TMEM (no smem traffic).
  // d = 64 : S_A[0,128) S_B[128,256) O_A[256,320) O_B[320,384) P_A[384,448) P_B[448,512)
  // d = 128: S_A[0,128) S_B[128,256) O_A[256,384) O_B[384,512); P_s aliases the first 64 cols of S_s
  // d = 128, BN = 64: S_A[0,64) S_B[64,128) P_A[128,160) P_B[160,192) O_A[256,384) O_B[384,512)
  static constexpr bool kPAlias = D == 128 && BN == 128;
  __device__ static constexpr uint32_t tS(int s) { return s * BN; }
  __device__ static constexpr uint32_t tO(int s) { return 256 + s * D; }
  __device__ static constexpr uint32_t tP(int s) {
    return kPAlias ? s * 128 + (SKR_FWD_SSPLIT ? 64 : 0) : (D == 128 ? 128 + s * 32 : 384 + s * 64);
  }
};

struct Bars {  // kUnits <= 8
  uint64_t q_full;
  uint64_t kv_full[8], kv_empty[8];
  uint64_t s_full[2], s_free[2], p_full[2], pv_done[2];
  uint64_t p_lo[2];   // kWG = 1: the first kSplitP / 8 of P is in TMEM (split P hand-over)
  uint32_t tmem_base;
};

// kWG = 1 (d = 128): the PV MMA of a tile is issued in two parts, keys [0, 16 kSplitP) as soon as
// the softmax has stored that much of P, the rest after the last quarter.
constexpr int kSplitP = 6;

// kPolyPer8: exponentials per 8 computed by ex2_poly on the FMA pipe.
// kWG: softmax warpgroups per head. 2: two warpgroups split the key columns of every row and combine
// their row maxima through shared memory (576 threads, <= 112 registers). 1 (d = 128 only): one
// warpgroup per head, thread = one full row of S (no cross-warpgroup exchange), P handed to the MMA in
// two parts (kSplitP) -- 320 threads, <= 200 registers.
// Softmax layout of the two-warpgroup-per-head kernel: 1 = row split (each warp owns 16 rows and all
// key columns, TMEM 16x256b loads, max / sum combined with shuffles); 0 = column split (each
// warpgroup owns half the key columns of all 128 rows, maxima exchanged through shared memory).
// Row split measured -4 to -6 % cycles at d = 128 (S4n1, C5n1) and -12 % at d = 64 (C2)
// (profiles/r02_experiments.md); the column split is kept as the documented alternative.

constexpr bool kRowSplit = SKR_FWD_ROWSPLIT;

template <int D, int kPolyPer8, int kWG = 2>
__global__ void __launch_bounds__((8 * kWG + 2) * 32, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, AttnArgs a, __nv_bfloat16* __restrict__ out,
                    float* __restrict__ lse, int pairs_per_group, int head_major) {
  using C = Cfg<D>;
  static_assert(kWG == 2 || (kWG == 1 && C::BN == 128), "one warpgroup per head: 128-key tiles");
  constexpr int kTmaW = 8 * kWG, kMmaW = 8 * kWG + 1, kSm = 128 * kWG;   // warp roles, softmax threads per head
  const int blk_pair = head_major ? blockIdx.y : blockIdx.x, blk_tile = head_major ? blockIdx.x : blockIdx.y;
  constexpr int BN = C::BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars* bars = reinterpret_cast<Bars*>(smem + C::kOffBar);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  // ---- work unit. d = 128: q-heads 2p and 2p + 1 of the whole head range -- with an odd GQA group
  // (Qwen: 7 q-heads per KV head) a pair may straddle two KV groups ("xg"); each head then has its
  // own K / V stream in the ring (units K_A K_B V_A V_B per KV tile instead of K V), so no CTA runs
  // a lone head (S4: fwd -2.5 %). d = 64: pairs within a group, the last one alone when the group is
  // odd (straddling pairs measured 6 % slower on C2: the ring then holds 1.5 tiles and the lone-head
  // CTAs are cheap when MUFU-bound).
  const int grp = a.hq / a.hkv;
  int ha, hb;
  if (pairs_per_group == 0) {
    ha = 2 * blk_pair;
    hb = (ha + 1 < a.hq) ? ha + 1 : -1;
  } else {
    const int g = blk_pair / pairs_per_group, p = blk_pair % pairs_per_group;
    ha = g * grp + 2 * p;
    hb = (2 * p + 1 < grp) ? ha + 1 : -1;
  }
  const int ga = ha / grp, gb = hb >= 0 ? hb / grp : ga;
  const bool xg = D == 128 && gb != ga;                // compile-time false for d = 64 (per-group pairs)
  const int U = xg ? 4 : 2;                             // ring units per KV tile
  const int seg = a.tiles[2 * blk_tile], tile = a.tiles[2 * blk_tile + 1];
  const int cu0 = a.cu[seg], cu1 = a.cu[seg + 1];
  const int r0 = cu0 + tile * BM;                       // first packed query row of the tile
  const int n_valid = min(BM, cu1 - r0);
  const int qp0 = a.q_pos[seg] + tile * BM;             // position of the tile's first query
  const int k_len = a.k_len[seg];                       // keys past k_len are invisible (ring CP)
  const int k_hi = min(qp0 + n_valid, k_len);           // keys visible to the last valid query
  const int n_kv = (max(k_hi, 0) + BN - 1) / BN;
  const int kst = a.k_start[seg];
  const int nq = hb >= 0 ? 2 : 1;
  if (n_kv == 0) {
    store_empty_tile<D>(a, out, lse, r0, n_valid, ha, nq);
    return;
  }

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    for (int u = 0; u < C::kUnits; ++u) mbar_init(&bars->kv_full[u], 1), mbar_init(&bars->kv_empty[u], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bars->s_full[s], 1);
      mbar_init(&bars->s_free[s], kSm);
      mbar_init(&bars->p_full[s], kSm);
      mbar_init(&bars->pv_done[s], 1);
      mbar_init(&bars->p_lo[s], kSm);
    }
    fence_mbar_init();
  }
  trace_init();
  if (warp == kMmaW) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == kTmaW) {
    // ================= TMA producer (warp-converged loop, one elected lane issues)
    if (elect_one()) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      mbar_expect_tx(&bars->q_full, nq * C::kQBytes);
      for (int s = 0; s < nq; ++s) {
        const int h = s == 0 ? ha : hb;
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_2d(smem + C::kOffQ + s * C::kQBytes + c * (BM * 128), &tm_q, &bars->q_full, h * D + c * 64, r0);
      }
    }
    __syncwarp();
    PhaseAcct pa;   // 0 waiting for a free unit, 1 issuing
    pa.start();
    int it = 0;
    for (int j = 0; j < n_kv; ++j) {
      for (int kv = 0; kv < U; ++kv, ++it) {
        const int u = it % C::kUnits;
        const bool is_k = xg ? kv < 2 : kv == 0;
        const int gg = (xg && (kv & 1)) ? gb : ga;
        pa.mark(1);
        mbar_wait_sleep(&bars->kv_empty[u], ((it / C::kUnits) & 1) ^ 1);
        pa.mark(0);
        if (lane == 0) trace(40 + (is_k ? 0 : 1), j);
        if (elect_one()) {
          mbar_expect_tx(&bars->kv_full[u], C::kKVBytes);
          uint8_t* dst = smem + C::kOffKV + u * C::kKVBytes;
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_2d(dst + c * (BN * 128), is_k ? &tm_k : &tm_v, &bars->kv_full[u], gg * D + c * 64,
                        kst + j * BN);
        }
        __syncwarp();
      }
    }
    pa.mark(1);
    if (lane == 0) pa.flush(g_trace_smem, kTmaW);
  } else if (warp == kMmaW) {
    // ================= MMA issuer: ONE elected thread runs the whole loop. Its waits spin on plain
    // try_wait (the suspend-hinted form measured 1.5 % slower here and 3 % faster in the backward,
    // profiles/r02_experiments.md). Measured (profiles/
    // umma_probe.py): the tensor pipe buffers only about one MMA ahead of the issuing thread, and
    // re-entering an elected region per MMA group costs ~200 cycles (R2UR of the descriptors,
    // BSSY/ELECT); inside a single elect.sync region groups + commits stream at the MMA floor.
    if (elect_one()) {
      const uint32_t id_s = idesc_bf16_f32(BM, BN, 0, 0);   // S = Q K^T   (both K-major)
      const uint32_t id_o = idesc_bf16_f32(BM, D, 0, 1);    // O += P V    (V is MN-major)
      const uint32_t sQ = smem_u32(smem + C::kOffQ), sKV = smem_u32(smem + C::kOffKV);
      // descriptor of (base + off) == descriptor of base + (off >> 4): the start address is the low field
      const uint64_t dq0 = sdesc_sw128(sQ, 16, 1024), dkv0 = sdesc_sw128(sKV, 16, 1024);
      const uint64_t dv0 = sdesc_sw128(sKV, BN * 128, 1024);
      auto issue_s = [&](int s, int u) {
        const uint64_t dq = dq0 + ((uint32_t)(s * C::kQBytes) >> 4), dk = dkv0 + ((uint32_t)(u * C::kKVBytes) >> 4);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = ((k / 4) * (BM * 128) + (k % 4) * 32) >> 4;
          const uint32_t koff = ((k / 4) * (BN * 128) + (k % 4) * 32) >> 4;
          umma_f16(tmem + C::tS(s), dq + off, dk + koff, id_s, k > 0);
        }
        umma_commit(&bars->s_full[s]);
      };
      // SKR_FWD_SSPLIT: one N = 64 half of S (keys / columns [64 h, 64 h + 64)); the caller commits
      const uint32_t id_s64 = idesc_bf16_f32(BM, 64, 0, 0);
      auto issue_s_half = [&](int s, int u, int h) {
        const uint64_t dq = dq0 + ((uint32_t)(s * C::kQBytes) >> 4);
        const uint64_t dk = dkv0 + ((uint32_t)(u * C::kKVBytes + h * 64 * 128) >> 4);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = ((k / 4) * (BM * 128) + (k % 4) * 32) >> 4;
          const uint32_t koff = ((k / 4) * (BN * 128) + (k % 4) * 32) >> 4;
          umma_f16(tmem + C::tS(s) + 64 * h, dq + off, dk + koff, id_s64, k > 0);
        }
      };
      // Row split with P aliasing S: the softmax never waits for an intermediate PV (s_full(j) implies
      // PV(j-1)), so pv_done is committed once, after the last PV (an arrive nobody waits for is what
      // compute-sanitizer's synccheck reports); its epilogue waits for phase 0
      constexpr bool kLastPvOnly = C::kPAlias && kRowSplit && kWG == 2;
      auto issue_pv = [&](int s, int u, bool acc, bool last = true) {
        const uint64_t dv = dv0 + ((uint32_t)(u * C::kKVBytes) >> 4);
#pragma unroll
        for (int k = 0; k < BN / 16; ++k)
          umma_f16_ts(tmem + C::tO(s), tmem + C::tP(s) + k * 8, dv + ((uint32_t)(k * 2048) >> 4), id_o, acc || k > 0);
        if (!kLastPvOnly || last) umma_commit(&bars->pv_done[s]);
      };
      // kWG = 1: PV in two parts, each waiting for its share of P (split hand-over)
      auto issue_pv_split = [&](int s, int u, bool acc, int jv) {
        const uint64_t dv = dv0 + ((uint32_t)(u * C::kKVBytes) >> 4);
        mbar_wait(&bars->p_lo[s], jv & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kSplitP; ++k)
          umma_f16_ts(tmem + C::tO(s), tmem + C::tP(s) + k * 8, dv + ((uint32_t)(k * 2048) >> 4), id_o, acc || k > 0);
        mbar_wait(&bars->p_full[s], jv & 1);
        tc_fence_after();
#pragma unroll
        for (int k = kSplitP; k < BN / 16; ++k)
          umma_f16_ts(tmem + C::tO(s), tmem + C::tP(s) + k * 8, dv + ((uint32_t)(k * 2048) >> 4), id_o, true);
        umma_commit(&bars->pv_done[s]);
      };
      mbar_wait_sleep(&bars->q_full, 0);
      tc_fence_after();
      // Static schedule with blocking waits (K/V units arrive in ring order K0 V0 K1 V1 ...). An
      // event-driven loop that polls every barrier was measured slower: with the tensor pipe only
      // ~one MMA ahead of the issuing thread, every poll between groups is pipe idle time.
      //  separate P (d=64):  [S_A(j) S_B(j)] release K(j); [PV_A(j-1) PV_B(j-1)] release V(j-1).
      //    S_s(j) waits until the softmax has read S_s(j-1) (s_free), so it overlaps softmax(j-1).
      //  P aliasing S (d=128): per head [PV_s(j-1) S_s(j)] back to back: S_s(j) overwrites P_s(j-1)
      //    after the in-order pipe has consumed it, and never queues behind the other head's PV.
      // ring position of head s's K / V unit of KV tile j (s ignored unless the pair straddles groups)
      auto kidx = [&](int j, int s) { return U * j + (xg ? s : 0); };
      auto vidx = [&](int j, int s) { return U * j + (xg ? 2 + s : 1); };
      auto kunit = [&](int j, int s) { return kidx(j, s) % C::kUnits; };
      auto vunit = [&](int j, int s) { return vidx(j, s) % C::kUnits; };
      const int nstream = xg ? 2 : 1;                     // distinct K (and V) units per KV tile
      PhaseAcct pa;   // 0 waiting for K, 1 for V, 2 for S free / P full, 3 issuing
      pa.start();
      auto wait_k = [&](int j) {
        pa.mark(3);
        for (int t = 0; t < nstream; ++t)
          mbar_wait(&bars->kv_full[kunit(j, t)], (kidx(j, t) / C::kUnits) & 1);
        pa.mark(0);
      };
      auto wait_v = [&](int j) {
        pa.mark(3);
        for (int t = 0; t < nstream; ++t)
          mbar_wait(&bars->kv_full[vunit(j, t)], (vidx(j, t) / C::kUnits) & 1);
        pa.mark(1);
      };
      auto free_k = [&](int j) {
        for (int t = 0; t < nstream; ++t) umma_commit(&bars->kv_empty[kunit(j, t)]);
      };
      auto free_v = [&](int j) {
        for (int t = 0; t < nstream; ++t) umma_commit(&bars->kv_empty[vunit(j, t)]);
      };
      if (!C::kPAlias && SKR_FWD_ORDER64 && kWG == 2) {
        // experiment (SKR_FWD_ORDER64): per head [S_s(j), PV_s(j-1)] instead of [S_A S_B][PV_A PV_B],
        // so head A's PV(j-1) never waits behind head B's s_free
        for (int j = 0; j <= n_kv; ++j) {
          if (j < n_kv) wait_k(j);
          if (j > 0) wait_v(j - 1);
          for (int s = 0; s < nq; ++s) {
            if (j < n_kv) {
              if (j > 0) mbar_wait(&bars->s_free[s], (j - 1) & 1);
              tc_fence_after();
              issue_s(s, kunit(j, s));
            }
            if (j > 0) {
              mbar_wait(&bars->p_full[s], (j - 1) & 1);
              tc_fence_after();
              issue_pv(s, vunit(j - 1, s), j - 1 > 0);
            }
          }
          if (j < n_kv) free_k(j);
          if (j > 0) free_v(j - 1);
        }
      } else if (!C::kPAlias) {
        for (int j = 0; j <= n_kv; ++j) {
          if (j < n_kv) {
            wait_k(j);
            for (int s = 0; s < nq; ++s) {
              pa.mark(3);
              if (j > 0) mbar_wait(&bars->s_free[s], (j - 1) & 1);
              pa.mark(2);
              tc_fence_after();
              trace(5 + s, j);
              issue_s(s, kunit(j, s));
              trace(1 + s, j);
            }
            free_k(j);   // K(j) free once every head's S MMAs completed
          }
          if (j > 0) {
            const int jv = j - 1;
            wait_v(jv);
            for (int s = 0; s < nq; ++s) {
              pa.mark(3);
              trace(7 + s, jv);
              if (kWG == 2) {
                mbar_wait(&bars->p_full[s], jv & 1);
                pa.mark(2);
                tc_fence_after();
                issue_pv(s, vunit(jv, s), jv > 0);
              } else {
                issue_pv_split(s, vunit(jv, s), jv > 0, jv);
                pa.mark(2);
              }
              trace(3 + s, jv);
            }
            free_v(jv);
          }
        }
      } else if (SKR_FWD_SSPLIT && kWG == 2 && kRowSplit) {
        wait_k(0);
        tc_fence_after();
        for (int s = 0; s < nq; ++s) issue_s(s, kunit(0, s));
        free_k(0);
        for (int j = 1; j <= n_kv; ++j) {
          const int jv = j - 1;
          wait_v(jv);
          if (j < n_kv) {
            wait_k(j);
            tc_fence_after();
          }
          for (int s = 0; s < nq; ++s) {
            if (j < n_kv) {   // the softmax has S_s(j-1) in registers: keys [0, 64) of S_s(j) may go in
              mbar_wait(&bars->p_lo[s], jv & 1);
              tc_fence_after();
              issue_s_half(s, kunit(j, s), 0);
            }
            mbar_wait(&bars->p_full[s], jv & 1);
            tc_fence_after();
            issue_pv(s, vunit(jv, s), jv > 0, j == n_kv);
            if (j < n_kv) {
              issue_s_half(s, kunit(j, s), 1);
              umma_commit(&bars->s_full[s]);
            }
          }
          free_v(jv);
          if (j < n_kv) free_k(j);
        }
      } else {
        wait_k(0);
        tc_fence_after();
        for (int s = 0; s < nq; ++s) issue_s(s, kunit(0, s));
        free_k(0);
        for (int j = 1; j <= n_kv; ++j) {
          const int jv = j - 1;
          wait_v(jv);
#if !SKR_FWD_PVFIRST
          if (j < n_kv) wait_k(j);
#endif
          for (int s = 0; s < nq; ++s) {
            pa.mark(3);
            if (kWG == 2) {
              mbar_wait(&bars->p_full[s], jv & 1);
              pa.mark(2);
              tc_fence_after();
              trace(7 + s, jv);
              issue_pv(s, vunit(jv, s), jv > 0, j == n_kv);
            } else {
              trace(7 + s, jv);
              issue_pv_split(s, vunit(jv, s), jv > 0, jv);
              pa.mark(2);
            }
#if SKR_FWD_PVFIRST
            if (s == 0 && j < n_kv) {   // PV_A(j-1) needs only V(j-1): issue it before K(j) lands
              wait_k(j);
              tc_fence_after();
            }
#endif
            if (j < n_kv) issue_s(s, kunit(j, s));
            trace(3 + s, jv);
          }
          free_v(jv);
          if (j < n_kv) free_k(j);
        }
      }
      pa.mark(3);
      pa.flush(g_trace_smem, kMmaW);
    }
    __syncwarp();
  } else if constexpr (kWG == 1) {
    // ================= softmax, one warpgroup per head: head s = warp / 4, thread = query row of the
    // tile holding all BN key columns (no cross-warpgroup maximum exchange). P (bf16 pairs) goes to
    // TMEM in four 32-key chunks; the MMA starts the PV of keys [0, 16 kSplitP) after the third
    // chunk (p_lo), the rest after the fourth (p_full). d = 128: P aliases S's first columns (already
    // in registers). d = 64: P has its own columns, so S_s(j+1) may be issued as soon as S_s(j) is
    // loaded (s_free), and P_s(j) is written only after PV_s(j-1) has read P_s(j-1).
    const int s = warp / 4;
    const int h = s == 0 ? ha : hb;
    if (h >= 0) {
      const int row = (warp % 4) * 32 + lane;
      const uint32_t lane_base = (uint32_t)((warp % 4) * 32) << 16;
      const uint32_t tS = tmem + lane_base + C::tS(s);
      const uint32_t tO = tmem + lane_base + C::tO(s);
      const uint32_t tP = tmem + lane_base + C::tP(s);
      const int qp = qp0 + row;
      const float sl2 = a.scale * 1.4426950408889634f;
      float m_ref = -INFINITY, l = 0.f;
      PhaseAcct pa;   // 0 wait S, 1 TMEM load S, 2 mask + max, 3 rescale O, 6 exps + store P
      pa.start();
      for (int j = 0; j < n_kv; ++j) {
        mbar_wait(&bars->s_full[s], j & 1);
        pa.mark(0);
        tc_fence_after();
        float x[BN];
        {
          uint32_t r[BN / 32][32];
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS + 32 * c, r[c]);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < BN / 32; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i) x[32 * c + i] = __uint_as_float(r[c][i]);
        }
        if (!C::kPAlias) {
          tc_fence_before();
          mbar_arrive(&bars->s_free[s]);      // S_s TMEM may now take S_s(j+1)
        }
        pa.mark(1);
        const int kv0 = j * BN;
        if (kv0 + BN - 1 > qp0 || kv0 + BN > k_len) {   // diagonal / last tile: mask keys after the query
#pragma unroll
          for (int i = 0; i < BN; ++i)
            if (kv0 + i > qp || kv0 + i >= k_len) x[i] = -INFINITY;
        }
        float mxs[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mxs[i] = x[i];
#pragma unroll
        for (int i = 8; i < BN; i += 16)
#pragma unroll
          for (int t = 0; t < 8; ++t) mxs[t] = fmax3(mxs[t], x[i + t], i + 8 + t < BN ? x[i + 8 + t] : x[i + t]);
        const float mx = fmaxf(fmaxf(fmaxf(mxs[0], mxs[1]), fmaxf(mxs[2], mxs[3])),
                               fmaxf(fmaxf(mxs[4], mxs[5]), fmaxf(mxs[6], mxs[7])));
        const float m_new = fmaxf(m_ref, mx * sl2);
        // tcgen05.ld/st are warp-collective: the lazy-rescale decision is made per warp
        const bool rescale = __any_sync(0xffffffffu, m_new > m_ref + kRescaleThreshold) || j == 0;
        const float alpha = (rescale && j > 0) ? ex2(m_ref - m_new) : 1.f;
        if (rescale) m_ref = m_new;
        const float neg_m = (m_ref == -INFINITY) ? 0.f : -m_ref;
        pa.mark(2);
        float2 ls2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 sl2_2 = make_float2(sl2, sl2), nm2 = make_float2(neg_m, neg_m);
        if (!C::kPAlias) {
          // exponentials first (registers: P packed, 64 words); P / O only after PV_s(j-1)
          uint32_t pk[BN / 2];
#pragma unroll
          for (int c = 0; c < BN; c += 8) {
            float pv[8];
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
              const float2 xx = ffma2(make_float2(x[c + i], x[c + i + 1]), sl2_2, nm2);
              pv[i] = i < kPolyPer8 ? ex2_poly(xx.x) : ex2(xx.x);
              pv[i + 1] = i + 1 < kPolyPer8 ? ex2_poly(xx.y) : ex2(xx.y);
              ls2[(i / 2) % 2] = fadd2(ls2[(i / 2) % 2], make_float2(pv[i], pv[i + 1]));
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) pk[c / 2 + i] = pack_bf16(pv[2 * i], pv[2 * i + 1]);
          }
          pa.mark(6);
          if (j > 0) {
            mbar_wait(&bars->pv_done[s], (j - 1) & 1);
            tc_fence_after();
          }
          if (rescale && j > 0) {
#pragma unroll
            for (int c = 0; c < D; c += 16) {
              uint32_t r[16];
              tmem_ld16(tO + c, r);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; i += 2) {
                const float2 v = fmul2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])),
                                       make_float2(alpha, alpha));
                r[i] = __float_as_uint(v.x), r[i + 1] = __float_as_uint(v.y);
              }
              tmem_st16(tO + c, r);
            }
          }
          pa.mark(3);
#pragma unroll
          for (int ch = 0; ch < BN / 32; ++ch) {
            uint32_t q16[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) q16[i] = pk[16 * ch + i];
            tmem_st16(tP + 16 * ch, q16);
            if (ch == kSplitP / 2 - 1) {
              tmem_wait_st();
              tc_fence_before();
              mbar_arrive(&bars->p_lo[s]);
            }
          }
          tmem_wait_st();
          tc_fence_before();
          mbar_arrive(&bars->p_full[s]);
          l = (rescale ? (j == 0 ? 0.f : l * alpha) : l) + ((ls2[0].x + ls2[0].y) + (ls2[1].x + ls2[1].y));
          pa.mark(4);
          continue;
        }
        if (rescale && j > 0) {
          // O_s must hold every PV up to j - 1 before it is scaled (S_s(j) completed after PV_s(j-1)
          // in the in-order pipe; the wait makes that explicit), and PV_s(j) only starts after p_lo
          mbar_wait(&bars->pv_done[s], (j - 1) & 1);
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D; c += 16) {
            uint32_t r[16];
            tmem_ld16(tO + c, r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              const float2 v = fmul2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])),
                                     make_float2(alpha, alpha));
              r[i] = __float_as_uint(v.x), r[i + 1] = __float_as_uint(v.y);
            }
            tmem_st16(tO + c, r);
          }
          tmem_wait_st();
        }
        pa.mark(3);
#pragma unroll
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 32; c += 8) {
            float pv[8];
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
              const float2 xx = ffma2(make_float2(x[32 * ch + c + i], x[32 * ch + c + i + 1]), sl2_2, nm2);
              pv[i] = i < kPolyPer8 ? ex2_poly(xx.x) : ex2(xx.x);
              pv[i + 1] = i + 1 < kPolyPer8 ? ex2_poly(xx.y) : ex2(xx.y);
              ls2[(i / 2) % 2] = fadd2(ls2[(i / 2) % 2], make_float2(pv[i], pv[i + 1]));
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) pk[c / 2 + i] = pack_bf16(pv[2 * i], pv[2 * i + 1]);
          }
          tmem_st16(tP + 16 * ch, pk);
          if (ch == kSplitP / 2 - 1) {          // keys [0, 16 kSplitP) of P are in TMEM
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&bars->p_lo[s]);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars->p_full[s]);
        l = (rescale ? (j == 0 ? 0.f : l * alpha) : l) + ((ls2[0].x + ls2[0].y) + (ls2[1].x + ls2[1].y));
        pa.mark(6);
      }
      if (lane == 0) pa.flush(g_trace_smem, warp);
      // ---- epilogue: O / l -> bf16 (all D columns of this row), LSE
      mbar_wait(&bars->pv_done[s], (n_kv - 1) & 1);
      tc_fence_after();
      const float inv_l = 1.f / l;
      const bool store = row < n_valid;
      __nv_bfloat16* orow = out + ((size_t)(r0 + row) * a.hq + h) * D;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        uint32_t r[32];
        tmem_ld32(tO + c, r);
        tmem_wait_ld();
        if (store) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(r[i + 0]) * inv_l, __uint_as_float(r[i + 1]) * inv_l);
            v.y = pack_bf16(__uint_as_float(r[i + 2]) * inv_l, __uint_as_float(r[i + 3]) * inv_l);
            v.z = pack_bf16(__uint_as_float(r[i + 4]) * inv_l, __uint_as_float(r[i + 5]) * inv_l);
            v.w = pack_bf16(__uint_as_float(r[i + 6]) * inv_l, __uint_as_float(r[i + 7]) * inv_l);
            *reinterpret_cast<uint4*>(orow + c + i) = v;
          }
        }
      }
      if (store) lse[(size_t)h * a.ld_lse + r0 + row] = (m_ref + __log2f(l)) * 0.6931471805599453f;
    }
  } else if constexpr (kRowSplit) {
    // ================= softmax, row split: head s = warp / 8; each of the head's 8 warps owns 16 query
    // rows (TMEM lanes 32 (warp % 4) + 16 ((warp / 4) % 2) + [0, 16)) and all BN key columns, read
    // with the 16x256b shape: thread t holds rows t/4 and t/4 + 8 of its 16, 32 key columns of each;
    // the four threads of a row combine its max (per tile) and sum (once) with two shuffles -- no
    // shared-memory exchange and no barrier between warps (the two-warpgroup column split needs both)
    const int s = warp / 8, hr = (warp / 4) % 2;
    const int h = s == 0 ? ha : hb;
    if (h >= 0) {
      const int lane0 = 32 * (warp % 4) + 16 * hr;            // this warp's first TMEM lane (= tile row)
      const uint32_t lane_base = (uint32_t)lane0 << 16;
      const uint32_t tS = tmem + lane_base + C::tS(s);
      const uint32_t tO = tmem + lane_base + C::tO(s);
      const uint32_t tP = tmem + lane_base + C::tP(s);
      const int rA = lane0 + lane / 4, rB = rA + 8;            // tile rows of this thread
      const int qA = qp0 + rA, qB = qp0 + rB;                  // their query positions
      const int cq = 2 * (lane % 4);                           // this thread's 2 columns of each group of 8
      const float sl2 = a.scale * 1.4426950408889634f;
      float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;   // l: this thread's partial row sums
      for (int j = 0; j < n_kv; ++j) {
        mbar_wait(&bars->s_full[s], j & 1);
        tc_fence_after();
        float x[BN / 2];
        {
          uint32_t r[BN / 2];
          tmem_ld16x256_x16(tS, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < BN / 2; ++i) x[i] = __uint_as_float(r[i]);
        }
        if (!C::kPAlias) {
          tc_fence_before();
          mbar_arrive(&bars->s_free[s]);      // S_s TMEM may now take S_s(j+1)
        } else if (SKR_FWD_SSPLIT && j + 1 < n_kv) {
          tc_fence_before();
          mbar_arrive(&bars->p_lo[s]);        // columns [0, 64) may take keys [0, 64) of S_s(j+1)
        }
        const int kv0 = j * BN;
        if (kv0 + BN - 1 > qp0 || kv0 + BN > k_len) {   // diagonal / last tile: mask keys after the query
#pragma unroll
          for (int k = 0; k < BN / 8; ++k)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int key = kv0 + 8 * k + cq + e;
              if (key > qA || key >= k_len) x[4 * k + e] = -INFINITY;
              if (key > qB || key >= k_len) x[4 * k + 2 + e] = -INFINITY;
            }
        }
        // row maxima: 4 independent fmax3 chains per row over this thread's 32 columns, then the row's
        // four threads (lanes 4i..4i+3) combine with two xor shuffles
        float ma[4], mb[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) ma[t] = x[4 * t], mb[t] = x[4 * t + 2];
#pragma unroll
        for (int k = 0; k < BN / 8; k += 4)
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            ma[t] = fmax3(ma[t], x[4 * (k + t) + 1], k + 4 < BN / 8 ? x[4 * (k + 4 + t)] : x[4 * (k + t) + 1]);
            mb[t] = fmax3(mb[t], x[4 * (k + t) + 3], k + 4 < BN / 8 ? x[4 * (k + 4 + t) + 2] : x[4 * (k + t) + 3]);
          }
        float mxA = fmaxf(fmaxf(ma[0], ma[1]), fmaxf(ma[2], ma[3]));
        float mxB = fmaxf(fmaxf(mb[0], mb[1]), fmaxf(mb[2], mb[3]));
        mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 1));
        mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 1));
        mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 2));
        mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 2));
        const float nA = fmaxf(mA, mxA * sl2), nB = fmaxf(mB, mxB * sl2);
        // tcgen05.ld/st are warp-collective: the lazy-rescale decision is made per warp (its 16 rows)
        const bool rescale =
            __any_sync(0xffffffffu, nA > mA + kRescaleThreshold || nB > mB + kRescaleThreshold) || j == 0;
        const float alA = (rescale && j > 0) ? ex2(mA - nA) : 1.f, alB = (rescale && j > 0) ? ex2(mB - nB) : 1.f;
        if (rescale) mA = nA, mB = nB;
        const float2 sl2_2 = make_float2(sl2, sl2);
        const float2 negA = make_float2(mA == -INFINITY ? 0.f : -mA, mA == -INFINITY ? 0.f : -mA);
        const float2 negB = make_float2(mB == -INFINITY ? 0.f : -mB, mB == -INFINITY ? 0.f : -mB);
        float2 sA = make_float2(0.f, 0.f), sB = make_float2(0.f, 0.f);
        uint32_t pk[BN / 4];
#pragma unroll
        for (int k = 0; k < BN / 8; ++k) {
          const float2 ea = ffma2(make_float2(x[4 * k], x[4 * k + 1]), sl2_2, negA);
          const float2 eb = ffma2(make_float2(x[4 * k + 2], x[4 * k + 3]), sl2_2, negB);
          // kPolyPer8 of every 8 exponentials on the FMA pipe (element index 4k + e within the thread)
          const int b = (4 * k) % 8;
          const float pa0 = b + 0 < kPolyPer8 ? ex2_poly(ea.x) : ex2(ea.x);
          const float pa1 = b + 1 < kPolyPer8 ? ex2_poly(ea.y) : ex2(ea.y);
          const float pb0 = b + 2 < kPolyPer8 ? ex2_poly(eb.x) : ex2(eb.x);
          const float pb1 = b + 3 < kPolyPer8 ? ex2_poly(eb.y) : ex2(eb.y);
          sA = fadd2(sA, make_float2(pa0, pa1));
          sB = fadd2(sB, make_float2(pb0, pb1));
          pk[2 * k] = pack_bf16(pa0, pa1);
          pk[2 * k + 1] = pack_bf16(pb0, pb1);
        }
        // PV_s(j-1) must have read P_s(j-1) and finished accumulating O_s before P / O are touched.
        // With P aliasing S (d = 128) that is implied by s_full(j): S_s(j) was issued after PV_s(j-1)
        // and the tensor pipe completes in order, so the wait (and its fence) is skipped.
        if (!C::kPAlias && j > 0) {
          mbar_wait(&bars->pv_done[s], (j - 1) & 1);
          tc_fence_after();
        }
        if (rescale && j > 0) {
#pragma unroll
          for (int c = 0; c < D; c += 32) {               // 32 columns (16 registers) at a time
            uint32_t o[16];
            tmem_ld16x256_x4(tO + c, o);
            tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const float2 va = fmul2(make_float2(__uint_as_float(o[4 * k]), __uint_as_float(o[4 * k + 1])),
                                      make_float2(alA, alA));
              const float2 vb = fmul2(make_float2(__uint_as_float(o[4 * k + 2]), __uint_as_float(o[4 * k + 3])),
                                      make_float2(alB, alB));
              o[4 * k] = __float_as_uint(va.x), o[4 * k + 1] = __float_as_uint(va.y);
              o[4 * k + 2] = __float_as_uint(vb.x), o[4 * k + 3] = __float_as_uint(vb.y);
            }
            tmem_st16x256_x4(tO + c, o);
          }
        }
        lA = (rescale ? (j == 0 ? 0.f : lA * alA) : lA) + (sA.x + sA.y);
        lB = (rescale ? (j == 0 ? 0.f : lB * alB) : lB) + (sB.x + sB.y);
        tmem_st16x128_x16(tP, pk);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars->p_full[s]);
      }
      // ---- epilogue: the row sums of the four threads of a row, O / l -> bf16, LSE
      lA += __shfl_xor_sync(0xffffffffu, lA, 1);
      lB += __shfl_xor_sync(0xffffffffu, lB, 1);
      lA += __shfl_xor_sync(0xffffffffu, lA, 2);
      lB += __shfl_xor_sync(0xffffffffu, lB, 2);
      mbar_wait(&bars->pv_done[s], C::kPAlias ? 0 : (n_kv - 1) & 1);   // kPAlias: one commit (the last PV)
      tc_fence_after();
      const float iA = 1.f / lA, iB = 1.f / lB;
      __nv_bfloat16* oA = out + ((size_t)(r0 + rA) * a.hq + h) * D + cq;
      __nv_bfloat16* oB = out + ((size_t)(r0 + rB) * a.hq + h) * D + cq;
#pragma unroll
      for (int c = 0; c < D; c += 32) {                    // 32 columns (16 registers) at a time
        uint32_t o[16];
        tmem_ld16x256_x4(tO + c, o);
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (rA < n_valid)
            *reinterpret_cast<uint32_t*>(oA + c + 8 * k) =
                pack_bf16(__uint_as_float(o[4 * k]) * iA, __uint_as_float(o[4 * k + 1]) * iA);
          if (rB < n_valid)
            *reinterpret_cast<uint32_t*>(oB + c + 8 * k) =
                pack_bf16(__uint_as_float(o[4 * k + 2]) * iB, __uint_as_float(o[4 * k + 3]) * iB);
        }
      }
      if (lane % 4 == 0) {
        if (rA < n_valid) lse[(size_t)h * a.ld_lse + r0 + rA] = (mA + __log2f(lA)) * 0.6931471805599453f;
        if (rB < n_valid) lse[(size_t)h * a.ld_lse + r0 + rB] = (mB + __log2f(lB)) * 0.6931471805599453f;
      }
    }
  } else {
    // ================= softmax: head s = warp / 8, key-column half hf = (warp / 4) % 2
    const int s = warp / 8, hf = (warp / 4) % 2;
    const int h = s == 0 ? ha : hb;
    if (h >= 0) {
      constexpr int HN = BN / 2;               // key columns of this half
      const int row = (warp % 4) * 32 + lane;  // TMEM lane == query row of the tile
      const uint32_t lane_base = (uint32_t)((warp % 4) * 32) << 16;
      const uint32_t tS = tmem + lane_base + C::tS(s) + hf * HN;
      const uint32_t tO = tmem + lane_base + C::tO(s) + hf * (D / 2);   // this half rescales / stores O[:, hf]
      const uint32_t tP = tmem + lane_base + C::tP(s) + hf * (HN / 2);
      float* red = reinterpret_cast<float*>(smem + C::kOffRed) + s * (2 * 2 * BM);   // [parity][half][row]
      const int qp = qp0 + row;                // this row's query position
      const float sl2 = a.scale * 1.4426950408889634f;
      float m_ref = -INFINITY, l = 0.f;
      PhaseAcct pa;   // 0 wait S, 1 TMEM load S, 2 mask + max + exchange, 3 wait PV, 4 rescale + store P, 6 exps
      pa.start();
      for (int j = 0; j < n_kv; ++j) {
        mbar_wait(&bars->s_full[s], j & 1);   // (a suspend-hinted wait measured the same, r02_run12)
        pa.mark(0);
        tc_fence_after();
        float x[HN];
        {
          uint32_t r[HN / 32][32];
#pragma unroll
          for (int c = 0; c < HN / 32; ++c) tmem_ld32(tS + 32 * c, r[c]);
          tmem_wait_ld();
#pragma unroll
          for (int c = 0; c < HN / 32; ++c)
#pragma unroll
            for (int i = 0; i < 32; ++i) x[32 * c + i] = __uint_as_float(r[c][i]);
        }
        if (!C::kPAlias) {
          tc_fence_before();
          mbar_arrive(&bars->s_free[s]);      // S_s TMEM may now take S_s(j+1)
        }
        pa.mark(1);
        const int kv0 = j * BN + hf * HN;
        if (kv0 + HN - 1 > qp0 || kv0 + HN > k_len) {   // diagonal / last tile: mask keys after the query
#pragma unroll
          for (int i = 0; i < HN; ++i)
            if (kv0 + i > qp || kv0 + i >= k_len) x[i] = -INFINITY;
        }
        // half-row max: 8 independent chains of three-input max, then combine with the other half
        float mxs[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) mxs[i] = x[i];
#pragma unroll
        for (int i = 8; i < HN; i += 16)
#pragma unroll
          for (int t = 0; t < 8; ++t) mxs[t] = fmax3(mxs[t], x[i + t], i + 8 + t < HN ? x[i + 8 + t] : x[i + t]);
        float mx = fmaxf(fmaxf(fmaxf(mxs[0], mxs[1]), fmaxf(mxs[2], mxs[3])),
                         fmaxf(fmaxf(mxs[4], mxs[5]), fmaxf(mxs[6], mxs[7])));
        float* rj = red + (j & 1) * (2 * BM);
        rj[hf * BM + row] = mx;
        tc_fence_before();                    // (d = 128) this half's S loads precede the partner's P stores
        named_bar_sync(1 + s, kSm);
        tc_fence_after();
        mx = fmaxf(mx, rj[(1 - hf) * BM + row]);
        const float m_new = fmaxf(m_ref, mx * sl2);
        pa.mark(2);
        // tcgen05.ld/st are warp-collective: the rescale decision is made per warp; the two halves of
        // a row see the same combined maximum, so their warps decide identically
        const bool rescale = __any_sync(0xffffffffu, m_new > m_ref + kRescaleThreshold) || j == 0;
        const float alpha = (rescale && j > 0) ? ex2(m_ref - m_new) : 1.f;
        if (rescale) m_ref = m_new;
        const float neg_m = (m_ref == -INFINITY) ? 0.f : -m_ref;
        float2 ls2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const float2 sl2_2 = make_float2(sl2, sl2), nm2 = make_float2(neg_m, neg_m);
        uint32_t pk[HN / 2];
#pragma unroll
        for (int c = 0; c < HN; c += 8) {
          float pv[8];
#pragma unroll
          for (int i = 0; i < 8; i += 2) {
            const float2 xx = ffma2(make_float2(x[c + i], x[c + i + 1]), sl2_2, nm2);
            // some exponentials on the FMA pipe, the rest on MUFU (MUFU ex2 is the d=64 bound)
            pv[i] = i < kPolyPer8 ? ex2_poly(xx.x) : ex2(xx.x);
            pv[i + 1] = i + 1 < kPolyPer8 ? ex2_poly(xx.y) : ex2(xx.y);
            ls2[(i / 2) % 2] = fadd2(ls2[(i / 2) % 2], make_float2(pv[i], pv[i + 1]));
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) pk[c / 2 + i] = pack_bf16(pv[2 * i], pv[2 * i + 1]);
        }
        const float ls[4] = {ls2[0].x, ls2[0].y, ls2[1].x, ls2[1].y};
        pa.mark(6);
        // PV_s(j-1) must have read P_s(j-1) and finished accumulating O_s before P / O are touched
        if (j > 0) {
          mbar_wait(&bars->pv_done[s], (j - 1) & 1);
          tc_fence_after();
        }
        pa.mark(3);
        if (rescale && j > 0) {
#pragma unroll
          for (int c = 0; c < D / 2; c += 16) {
            uint32_t r[16];
            tmem_ld16(tO + c, r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              const float2 v = fmul2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])),
                                     make_float2(alpha, alpha));
              r[i] = __float_as_uint(v.x), r[i + 1] = __float_as_uint(v.y);
            }
            tmem_st16(tO + c, r);
          }
        }
        l = (rescale ? (j == 0 ? 0.f : l * alpha) : l) + ((ls[0] + ls[1]) + (ls[2] + ls[3]));
        tmem_st_half<HN / 2>(tP, pk);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bars->p_full[s]);
        pa.mark(4);
      }
      if (lane == 0) pa.flush(g_trace_smem, warp);
      // ---- epilogue: combine the halves' row sums, O / l -> bf16 (this half's d columns), LSE
      float* lr = red + (n_kv & 1) * (2 * BM);   // a parity slot no half reads any more
      lr[hf * BM + row] = l;
      named_bar_sync(1 + s, kSm);
      l += lr[(1 - hf) * BM + row];
      mbar_wait(&bars->pv_done[s], (n_kv - 1) & 1);
      tc_fence_after();
      const float inv_l = 1.f / l;
      const bool store = row < n_valid;
      __nv_bfloat16* orow = out + ((size_t)(r0 + row) * a.hq + h) * D + hf * (D / 2);
#pragma unroll
      for (int c = 0; c < D / 2; c += 32) {
        uint32_t r[32];
        tmem_ld32(tO + c, r);
        tmem_wait_ld();
        if (store) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) {
            uint4 v;
            v.x = pack_bf16(__uint_as_float(r[i + 0]) * inv_l, __uint_as_float(r[i + 1]) * inv_l);
            v.y = pack_bf16(__uint_as_float(r[i + 2]) * inv_l, __uint_as_float(r[i + 3]) * inv_l);
            v.z = pack_bf16(__uint_as_float(r[i + 4]) * inv_l, __uint_as_float(r[i + 5]) * inv_l);
            v.w = pack_bf16(__uint_as_float(r[i + 6]) * inv_l, __uint_as_float(r[i + 7]) * inv_l);
            *reinterpret_cast<uint4*>(orow + c + i) = v;
          }
        }
      }
      if (store && hf == 0) lse[(size_t)h * a.ld_lse + r0 + row] = (m_ref + __log2f(l)) * 0.6931471805599453f;
    }
    }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaW) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------------------------------------
// d = 128, one q-head per CTA ("1h"): TMEM S0 [0,128) S1 [128,256) P [256,320) O [384,512). With
// one head the S accumulator can be DOUBLE-buffered and P gets its own columns, so S(j+1) is
// computed while the softmax works on S(j) and PV(j) overlaps the exponentials of j+1 -- the
// two-head kernel's per-head chain S(j) -> softmax -> PV(j) -> S(j+1) (P aliasing S) is gone.
// Four softmax warpgroups split the 128 key columns (32 each) and combine row maxima through smem.
// The cost: K/V tiles are loaded and read per head (no GQA sharing inside the CTA).
struct Cfg1h {
  static constexpr int D = 128, kChunks = 2;
  static constexpr int kQBytes = BM * D * 2, kKVBytes = 128 * D * 2;
  static constexpr int kUnits = 5;
  static constexpr int kOffQ = 0, kOffKV = kQBytes;
  static constexpr int kOffRed = kOffKV + kUnits * kKVBytes;        // [parity][4][BM] maxima, then [4][BM] sums
  static constexpr int kOffBar = kOffRed + (2 * 4 + 4) * BM * 4;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static constexpr uint32_t tS(int b) { return b * 128; }
  static constexpr uint32_t tP = 256, tO = 384;
};

struct Bars1h {
  uint64_t q_full;
  uint64_t kv_full[8], kv_empty[8];
  uint64_t s_full[2], s_free[2], p_full, pv_done;
  uint32_t tmem_base;
};

template <int kPolyPer8>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd1h_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                      const __grid_constant__ CUtensorMap tm_v, AttnArgs a, __nv_bfloat16* __restrict__ out,
                      float* __restrict__ lse) {
  using C = Cfg1h;
  constexpr int D = 128, BN = 128, HN = 32;            // key columns per softmax warpgroup
  constexpr int kSm = 4 * 128;                         // softmax threads of the head
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars1h* bars = reinterpret_cast<Bars1h*>(smem + C::kOffBar);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  const int h = blockIdx.x, g = h / (a.hq / a.hkv);
  const int seg = a.tiles[2 * blockIdx.y], tile = a.tiles[2 * blockIdx.y + 1];
  const int cu0 = a.cu[seg], cu1 = a.cu[seg + 1];
  const int r0 = cu0 + tile * BM;
  const int n_valid = min(BM, cu1 - r0);
  const int qp0 = a.q_pos[seg] + tile * BM;
  const int k_len = a.k_len[seg];
  const int n_kv = (max(min(qp0 + n_valid, k_len), 0) + BN - 1) / BN;
  const int kst = a.k_start[seg];
  if (n_kv == 0) {
    store_empty_tile<128>(a, out, lse, r0, n_valid, h, 1);
    return;
  }

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    for (int u = 0; u < C::kUnits; ++u) mbar_init(&bars->kv_full[u], 1), mbar_init(&bars->kv_empty[u], 1);
    for (int b = 0; b < 2; ++b) mbar_init(&bars->s_full[b], 1), mbar_init(&bars->s_free[b], kSm);
    mbar_init(&bars->p_full, kSm);
    mbar_init(&bars->pv_done, 1);
    fence_mbar_init();
  }
  if (warp == kMmaWarp) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == kTmaWarp) {
    if (elect_one()) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      mbar_expect_tx(&bars->q_full, C::kQBytes);
      for (int c = 0; c < C::kChunks; ++c)
        tma_load_2d(smem + C::kOffQ + c * (BM * 128), &tm_q, &bars->q_full, h * D + c * 64, r0);
    }
    __syncwarp();
    int it = 0;
    for (int j = 0; j < n_kv; ++j) {
      for (int kv = 0; kv < 2; ++kv, ++it) {
        const int u = it % C::kUnits;
        mbar_wait_sleep(&bars->kv_empty[u], ((it / C::kUnits) & 1) ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&bars->kv_full[u], C::kKVBytes);
          uint8_t* dst = smem + C::kOffKV + u * C::kKVBytes;
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_2d(dst + c * (BN * 128), kv == 0 ? &tm_k : &tm_v, &bars->kv_full[u], g * D + c * 64,
                        kst + j * BN);
        }
        __syncwarp();
      }
    }
  } else if (warp == kMmaWarp) {
    if (elect_one()) {
      const uint32_t id_s = idesc_bf16_f32(BM, BN, 0, 0), id_o = idesc_bf16_f32(BM, D, 0, 1);
      const uint64_t dq0 = sdesc_sw128(smem_u32(smem + C::kOffQ), 16, 1024);
      const uint64_t dkv0 = sdesc_sw128(smem_u32(smem + C::kOffKV), 16, 1024);
      const uint64_t dv0 = sdesc_sw128(smem_u32(smem + C::kOffKV), BN * 128, 1024);
      auto kunit = [&](int j) { return (2 * j) % C::kUnits; };
      auto vunit = [&](int j) { return (2 * j + 1) % C::kUnits; };
      mbar_wait_sleep(&bars->q_full, 0);
      tc_fence_after();
      // S(j) into buffer j & 1 as soon as K(j) is in and the softmax has read S(j-2); then PV(j-1)
      // once P(j-1) is stored: S(j) overlaps softmax(j-1), PV(j-1) overlaps the exps of j
      for (int j = 0; j <= n_kv; ++j) {
        if (j < n_kv) {
          mbar_wait_sleep(&bars->kv_full[kunit(j)], ((2 * j) / C::kUnits) & 1);
          if (j >= 2) mbar_wait_sleep(&bars->s_free[j & 1], ((j - 2) >> 1) & 1);
          tc_fence_after();
          const uint64_t dk = dkv0 + ((uint32_t)(kunit(j) * C::kKVBytes) >> 4);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = ((k / 4) * (BM * 128) + (k % 4) * 32) >> 4;
            const uint32_t koff = ((k / 4) * (BN * 128) + (k % 4) * 32) >> 4;
            umma_f16(tmem + C::tS(j & 1), dq0 + off, dk + koff, id_s, k > 0);
          }
          umma_commit(&bars->s_full[j & 1]);
          umma_commit(&bars->kv_empty[kunit(j)]);
        }
        if (j > 0) {
          const int jv = j - 1;
          mbar_wait_sleep(&bars->kv_full[vunit(jv)], ((2 * jv + 1) / C::kUnits) & 1);
          mbar_wait_sleep(&bars->p_full, jv & 1);
          tc_fence_after();
          const uint64_t dv = dv0 + ((uint32_t)(vunit(jv) * C::kKVBytes) >> 4);
#pragma unroll
          for (int k = 0; k < BN / 16; ++k)
            umma_f16_ts(tmem + C::tO, tmem + C::tP + k * 8, dv + ((uint32_t)(k * 2048) >> 4), id_o, jv > 0 || k > 0);
          umma_commit(&bars->pv_done);
          umma_commit(&bars->kv_empty[vunit(jv)]);
        }
      }
    }
    __syncwarp();
  } else {
    const int w = warp / 4;                  // key-column quarter [32w, 32w + 32)
    const int row = (warp % 4) * 32 + lane;
    const uint32_t lane_base = (uint32_t)((warp % 4) * 32) << 16;
    const uint32_t tO = tmem + lane_base + C::tO + w * (D / 4);
    const uint32_t tP = tmem + lane_base + C::tP + w * (HN / 2);
    float* red = reinterpret_cast<float*>(smem + C::kOffRed);           // [parity][4][BM]
    float* lsum = red + 2 * 4 * BM;                                     // [4][BM]
    const int qp = qp0 + row;
    const float sl2 = a.scale * 1.4426950408889634f;
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      mbar_wait(&bars->s_full[b], (j >> 1) & 1);
      tc_fence_after();
      float x[HN];
      {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + C::tS(b) + w * HN, r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) x[i] = __uint_as_float(r[i]);
      }
      tc_fence_before();
      mbar_arrive(&bars->s_free[b]);          // S buffer b may take S(j + 2)
      const int kv0 = j * BN + w * HN;
      if (kv0 + HN - 1 > qp0 || kv0 + HN > k_len) {
#pragma unroll
        for (int i = 0; i < HN; ++i)
          if (kv0 + i > qp || kv0 + i >= k_len) x[i] = -INFINITY;
      }
      float mxs[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mxs[i] = fmax3(x[i], x[i + 8], x[i + 16]);
#pragma unroll
      for (int i = 0; i < 8; ++i) mxs[i] = fmaxf(mxs[i], x[i + 24]);
      float mx = fmaxf(fmaxf(fmaxf(mxs[0], mxs[1]), fmaxf(mxs[2], mxs[3])),
                       fmaxf(fmaxf(mxs[4], mxs[5]), fmaxf(mxs[6], mxs[7])));
      float* rj = red + b * (4 * BM);
      rj[w * BM + row] = mx;
      named_bar_sync(1, kSm);
      mx = fmaxf(fmaxf(rj[row], rj[BM + row]), fmaxf(rj[2 * BM + row], rj[3 * BM + row]));
      const float m_new = fmaxf(m_ref, mx * sl2);
      const bool rescale = __any_sync(0xffffffffu, m_new > m_ref + kRescaleThreshold) || j == 0;
      const float alpha = (rescale && j > 0) ? ex2(m_ref - m_new) : 1.f;
      if (rescale) m_ref = m_new;
      const float neg_m = (m_ref == -INFINITY) ? 0.f : -m_ref;
      float2 ls2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const float2 sl2_2 = make_float2(sl2, sl2), nm2 = make_float2(neg_m, neg_m);
      uint32_t pk[HN / 2];
#pragma unroll
      for (int c = 0; c < HN; c += 8) {
        float pv[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float2 xx = ffma2(make_float2(x[c + i], x[c + i + 1]), sl2_2, nm2);
          pv[i] = i < kPolyPer8 ? ex2_poly(xx.x) : ex2(xx.x);
          pv[i + 1] = i + 1 < kPolyPer8 ? ex2_poly(xx.y) : ex2(xx.y);
          ls2[(i / 2) % 2] = fadd2(ls2[(i / 2) % 2], make_float2(pv[i], pv[i + 1]));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) pk[c / 2 + i] = pack_bf16(pv[2 * i], pv[2 * i + 1]);
      }
      // PV(j-1) must have consumed P and finished accumulating O before P / O are touched
      if (j > 0) {
        mbar_wait(&bars->pv_done, (j - 1) & 1);
        tc_fence_after();
      }
      if (rescale && j > 0) {
#pragma unroll
        for (int c = 0; c < D / 4; c += 16) {
          uint32_t r[16];
          tmem_ld16(tO + c, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float2 v = fmul2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])),
                                   make_float2(alpha, alpha));
            r[i] = __float_as_uint(v.x), r[i + 1] = __float_as_uint(v.y);
          }
          tmem_st16(tO + c, r);
        }
      }
      l = (rescale ? (j == 0 ? 0.f : l * alpha) : l) + ((ls2[0].x + ls2[0].y) + (ls2[1].x + ls2[1].y));
      tmem_st16(tP, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars->p_full);
    }
    // epilogue: combine the quarters' row sums, O / l -> bf16 (this quarter's 32 d columns), LSE
    lsum[w * BM + row] = l;
    named_bar_sync(1, kSm);
    l = (lsum[row] + lsum[BM + row]) + (lsum[2 * BM + row] + lsum[3 * BM + row]);
    mbar_wait(&bars->pv_done, (n_kv - 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l;
    uint32_t r[32];
    tmem_ld32(tO, r);
    tmem_wait_ld();
    if (row < n_valid) {
      __nv_bfloat16* orow = out + ((size_t)(r0 + row) * a.hq + h) * D + w * (D / 4);
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 v;
        v.x = pack_bf16(__uint_as_float(r[i + 0]) * inv_l, __uint_as_float(r[i + 1]) * inv_l);
        v.y = pack_bf16(__uint_as_float(r[i + 2]) * inv_l, __uint_as_float(r[i + 3]) * inv_l);
        v.z = pack_bf16(__uint_as_float(r[i + 4]) * inv_l, __uint_as_float(r[i + 5]) * inv_l);
        v.w = pack_bf16(__uint_as_float(r[i + 6]) * inv_l, __uint_as_float(r[i + 7]) * inv_l);
        *reinterpret_cast<uint4*>(orow + i) = v;
      }
      if (w == 0) lse[(size_t)h * a.ld_lse + r0 + row] = (m_ref + __log2f(l)) * 0.6931471805599453f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc<512>(tmem);
}


// ---------------------------------------------------------------------------------------------
// d = 128, one q-head per CTA PAIR ("2sm", cta_group::2, opt-in SKR_FWD_2SM=1): the cluster's two
// CTAs take query tiles 2t and 2t + 1 of one segment (a 256-row super tile of the work list) and
// run one M = 256 MMA stream issued by the leader.
// Each CTA holds its 128 Q rows, HALF of every K tile (64 keys: S's B operand is split by N) and
// HALF of every V tile (64 of the d columns: PV's B operand), so per CTA the shared-memory operand
// and TMA bytes per KV tile are 96 KB instead of the 1h kernel's 160 KB, with the 1h kernel's
// double-buffered S and separate P (TMEM S0 [0,128) S1 [128,256) P [256,320) O [384,512) in BOTH
// CTAs). Hand-overs: TMA completions and the softmax's s_free / p_full arrivals of both CTAs land
// on the leader's barriers (shared::cluster addresses); the leader's commits multicast to both.
struct Cfg2sm {
  static constexpr int D = 128;
  static constexpr int kQBytes = BM * D * 2;                 // this CTA's 128 query rows
  static constexpr int kKVBytes = 16384;                     // K: 64 keys x 128 d; V: 128 keys x 64 d
  static constexpr int kUnits = 8;
  static constexpr int kOffQ = 0, kOffKV = kQBytes;
  static constexpr int kOffRed = kOffKV + kUnits * kKVBytes;
  static constexpr int kOffBar = kOffRed + (2 * 4 + 4) * BM * 4;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  static constexpr uint32_t tS(int b) { return b * 128; }
  static constexpr uint32_t tP(int b) { return 256 + b * 64; }   // P double-buffered: P(j) may be
  static constexpr uint32_t tO = 384;                            // stored while PV(j - 1) runs
};

struct Bars2sm {
  uint64_t q_full;
  uint64_t kv_full[8], kv_empty[8];
  uint64_t s_full[2], s_free[2], p_full[2], pv_done[2];
  uint32_t tmem_base;
};

template <int kPolyPer8>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(320, 1)
    attn_fwd2sm_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                       const __grid_constant__ CUtensorMap tm_v, AttnArgs a, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ lse) {
  using C = Cfg2sm;
  constexpr int D = 128, BN = 128, HN = 64;            // key columns per softmax warpgroup (two halves)
  constexpr int kSm = 2 * 128;
  constexpr int kTma = 8, kMma = 9;
  constexpr int kArrivals = 2 * 8;                     // s_free / p_full: one per softmax warp of both CTAs
  // work list entries are 256-row super tiles (skr_attn_block_m = 256 in this mode): CTA r of the
  // pair takes the super tile's 128-row tile 2t + r
  const int seg = a.tiles[2 * blockIdx.y], tile0 = 2 * a.tiles[2 * blockIdx.y + 1];
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars2sm* bars = reinterpret_cast<Bars2sm*>(smem + C::kOffBar);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;

  const int h = blockIdx.x >> 1, g = h / (a.hq / a.hkv);
  const int cu0 = a.cu[seg], cu1 = a.cu[seg + 1];
  const int rs0 = cu0 + tile0 * BM;                     // first row of the super tile
  const int n_valid_pair = min(2 * BM, cu1 - rs0);
  const int k_len = a.k_len[seg];
  const int n_kv = (max(min(a.q_pos[seg] + tile0 * BM + n_valid_pair, k_len), 0) + BN - 1) / BN;   // same in both CTAs
  const int r0 = rs0 + (int)rank * BM;                  // this CTA's rows
  const int n_valid = min(BM, cu1 - r0);               // may be <= 0 for rank 1
  const int qp0 = a.q_pos[seg] + (tile0 + (int)rank) * BM;
  const int kst = a.k_start[seg];
  if (n_kv == 0) {                                      // both CTAs of the pair (n_kv is shared)
    store_empty_tile<128>(a, out, lse, r0, max(n_valid, 0), h, 1);
    return;
  }

  if (threadIdx.x == 0) {
    mbar_init(&bars->q_full, 1);
    for (int u = 0; u < C::kUnits; ++u) mbar_init(&bars->kv_full[u], 1), mbar_init(&bars->kv_empty[u], 1);
    for (int b = 0; b < 2; ++b) mbar_init(&bars->s_full[b], 1), mbar_init(&bars->s_free[b], kArrivals);
    for (int b = 0; b < 2; ++b) mbar_init(&bars->p_full[b], kArrivals), mbar_init(&bars->pv_done[b], 1);
    fence_mbar_init();
  }
  if (warp == kMma) tmem_alloc_pair<512>(&bars->tmem_base);
  tc_fence_before();
  cluster_sync_all();                                   // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == kTma) {
    const uint32_t q_full_l = mapa_shared(&bars->q_full, 0);
    if (elect_one()) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      if (leader) mbar_expect_tx(&bars->q_full, 2 * C::kQBytes);
      for (int c = 0; c < 2; ++c)
        tma_load_2d_pair(smem + C::kOffQ + c * (BM * 128), &tm_q, q_full_l, h * D + c * 64, r0);
    }
    __syncwarp();
    int it = 0;
    for (int j = 0; j < n_kv; ++j) {
      for (int kv = 0; kv < 2; ++kv, ++it) {
        const int u = it % C::kUnits;
        mbar_wait_sleep(&bars->kv_empty[u], ((it / C::kUnits) & 1) ^ 1);
        if (elect_one()) {
          if (leader) mbar_expect_tx(&bars->kv_full[u], 2 * C::kKVBytes);
          const uint32_t full_l = mapa_shared(&bars->kv_full[u], 0);
          uint8_t* dst = smem + C::kOffKV + u * C::kKVBytes;
          if (kv == 0) {   // K rows [64 rank, 64 rank + 64) of the tile, both 64-column chunks of d
            for (int c = 0; c < 2; ++c)
              tma_load_2d_pair(dst + c * (64 * 128), &tm_k, full_l, g * D + c * 64, kst + j * BN + 64 * (int)rank);
          } else {         // V: all 128 keys, d columns [64 rank, 64 rank + 64)
            tma_load_2d_pair(dst, &tm_v, full_l, g * D + 64 * (int)rank, kst + j * BN);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp == kMma) {
    if (leader && elect_one()) {
      const uint32_t id_s = idesc_bf16_f32(2 * BM, BN, 0, 0), id_o = idesc_bf16_f32(2 * BM, D, 0, 1);
      const uint64_t dq0 = sdesc_sw128(smem_u32(smem + C::kOffQ), 16, 1024);
      const uint64_t dkv0 = sdesc_sw128(smem_u32(smem + C::kOffKV), 16, 1024);
      const uint64_t dv0 = sdesc_sw128(smem_u32(smem + C::kOffKV), 128 * 128, 1024);
      auto kunit = [&](int j) { return (2 * j) % C::kUnits; };
      auto vunit = [&](int j) { return (2 * j + 1) % C::kUnits; };
      mbar_wait_sleep(&bars->q_full, 0);
      tc_fence_after();
      for (int j = 0; j <= n_kv; ++j) {
        if (j < n_kv) {
          mbar_wait_sleep(&bars->kv_full[kunit(j)], ((2 * j) / C::kUnits) & 1);
          if (j >= 2) mbar_wait_sleep(&bars->s_free[j & 1], ((j - 2) >> 1) & 1);
          tc_fence_after();
          const uint64_t dk = dkv0 + ((uint32_t)(kunit(j) * C::kKVBytes) >> 4);
#pragma unroll
          for (int k = 0; k < D / 16; ++k) {
            const uint32_t off = ((k / 4) * (BM * 128) + (k % 4) * 32) >> 4;
            const uint32_t koff = ((k / 4) * (64 * 128) + (k % 4) * 32) >> 4;
            umma2_f16(tmem + C::tS(j & 1), dq0 + off, dk + koff, id_s, k > 0);
          }
          umma2_commit_both(&bars->s_full[j & 1]);
          umma2_commit_both(&bars->kv_empty[kunit(j)]);
        }
        if (j > 0) {
          const int jv = j - 1;
          mbar_wait_sleep(&bars->kv_full[vunit(jv)], ((2 * jv + 1) / C::kUnits) & 1);
          mbar_wait_sleep(&bars->p_full[jv & 1], (jv >> 1) & 1);
          tc_fence_after();
          const uint64_t dv = dv0 + ((uint32_t)(vunit(jv) * C::kKVBytes) >> 4);
#pragma unroll
          for (int k = 0; k < BN / 16; ++k)
            umma2_f16_ts(tmem + C::tO, tmem + C::tP(jv & 1) + k * 8, dv + ((uint32_t)(k * 2048) >> 4), id_o,
                         jv > 0 || k > 0);
          umma2_commit_both(&bars->pv_done[jv & 1]);
          umma2_commit_both(&bars->kv_empty[vunit(jv)]);
        }
      }
    }
    __syncwarp();
  } else {
    const int w = warp / 4;                  // key-column half [64w, 64w + 64)
    const int row = (warp % 4) * 32 + lane;
    const uint32_t lane_base = (uint32_t)((warp % 4) * 32) << 16;
    const uint32_t tO = tmem + lane_base + C::tO + w * (D / 2);
    const uint32_t tP0 = tmem + lane_base + C::tP(0) + w * (HN / 2);
    const uint32_t s_free_l[2] = {mapa_shared(&bars->s_free[0], 0), mapa_shared(&bars->s_free[1], 0)};
    const uint32_t p_full_l[2] = {mapa_shared(&bars->p_full[0], 0), mapa_shared(&bars->p_full[1], 0)};
    const uint32_t red = smem_u32(smem + C::kOffRed);                 // [parity][2][BM] maxima, [2][BM] sums
    const int qp = qp0 + row;
    const float sl2 = a.scale * 1.4426950408889634f;
    float m_ref = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int b = j & 1;
      mbar_wait(&bars->s_full[b], (j >> 1) & 1);
      tc_fence_after();
      float x[HN];
      {
        uint32_t r[2][32];
        tmem_ld32(tmem + lane_base + C::tS(b) + w * HN, r[0]);
        tmem_ld32(tmem + lane_base + C::tS(b) + w * HN + 32, r[1]);
        tmem_wait_ld();
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
          for (int i = 0; i < 32; ++i) x[32 * c + i] = __uint_as_float(r[c][i]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(s_free_l[b]);   // S buffer b may take S(j + 2)
      const int kv0 = j * BN + w * HN;
      if (kv0 + HN - 1 > qp0 || kv0 + HN > k_len) {
#pragma unroll
        for (int i = 0; i < HN; ++i)
          if (kv0 + i > qp || kv0 + i >= k_len) x[i] = -INFINITY;
      }
      float mxs[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mxs[i] = x[i];
#pragma unroll
      for (int i = 8; i < HN; i += 16)
#pragma unroll
        for (int t = 0; t < 8; ++t) mxs[t] = fmax3(mxs[t], x[i + t], i + 8 + t < HN ? x[i + 8 + t] : x[i + t]);
      float mx = fmaxf(fmaxf(fmaxf(mxs[0], mxs[1]), fmaxf(mxs[2], mxs[3])),
                       fmaxf(fmaxf(mxs[4], mxs[5]), fmaxf(mxs[6], mxs[7])));
      const uint32_t rj = red + 4 * (b * 2 * BM);
      st_shared_f32(rj + 4 * (w * BM + row), mx);
      named_bar_sync(1, kSm);
      mx = fmaxf(mx, ld_shared_f32(rj + 4 * ((1 - w) * BM + row)));
      const float m_new = fmaxf(m_ref, mx * sl2);
      const bool rescale = __any_sync(0xffffffffu, m_new > m_ref + kRescaleThreshold) || j == 0;
      const float alpha = (rescale && j > 0 && m_ref != -INFINITY) ? ex2(m_ref - m_new) : 1.f;
      if (rescale) m_ref = m_new;
      const float neg_m = (m_ref == -INFINITY) ? 0.f : -m_ref;
      float2 ls2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const float2 sl2_2 = make_float2(sl2, sl2), nm2 = make_float2(neg_m, neg_m);
      uint32_t pk[HN / 2];
#pragma unroll
      for (int c = 0; c < HN; c += 8) {
        float pv[8];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float2 xx = ffma2(make_float2(x[c + i], x[c + i + 1]), sl2_2, nm2);
          pv[i] = i < kPolyPer8 ? ex2_poly(xx.x) : ex2(xx.x);
          pv[i + 1] = i + 1 < kPolyPer8 ? ex2_poly(xx.y) : ex2(xx.y);
          ls2[(i / 2) % 2] = fadd2(ls2[(i / 2) % 2], make_float2(pv[i], pv[i + 1]));
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) pk[c / 2 + i] = pack_bf16(pv[2 * i], pv[2 * i + 1]);
      }
      // P buffer j & 1 is free once PV(j - 2) has read it; O may be rescaled only once PV(j - 1)
      // has accumulated into it (rare: lazy rescale)
      if (j >= 2) mbar_wait(&bars->pv_done[b], ((j - 2) >> 1) & 1);
      if (rescale && j > 0) mbar_wait(&bars->pv_done[b ^ 1], ((j - 1) >> 1) & 1);
      tc_fence_after();
      if (rescale && j > 0) {
#pragma unroll
        for (int c = 0; c < D / 2; c += 16) {
          uint32_t r[16];
          tmem_ld16(tO + c, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 16; i += 2) {
            const float2 v = fmul2(make_float2(__uint_as_float(r[i]), __uint_as_float(r[i + 1])),
                                   make_float2(alpha, alpha));
            r[i] = __float_as_uint(v.x), r[i + 1] = __float_as_uint(v.y);
          }
          tmem_st16(tO + c, r);
        }
      }
      l = (rescale ? (j == 0 ? 0.f : l * alpha) : l) + ((ls2[0].x + ls2[0].y) + (ls2[1].x + ls2[1].y));
      tmem_st32(tP0 + b * 64, pk);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(p_full_l[b]);
    }
    const uint32_t lsum = red + 4 * (2 * 2 * BM);
    st_shared_f32(lsum + 4 * (w * BM + row), l);
    named_bar_sync(1, kSm);
    l += ld_shared_f32(lsum + 4 * ((1 - w) * BM + row));
    mbar_wait(&bars->pv_done[(n_kv - 1) & 1], ((n_kv - 1) >> 1) & 1);
    tc_fence_after();
    const float inv_l = 1.f / l;
#pragma unroll
    for (int c = 0; c < D / 2; c += 32) {
      uint32_t r[32];
      tmem_ld32(tO + c, r);
      tmem_wait_ld();
      if (row < n_valid) {
        __nv_bfloat16* orow = out + ((size_t)(r0 + row) * a.hq + h) * D + w * (D / 2) + c;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 v;
          v.x = pack_bf16(__uint_as_float(r[i + 0]) * inv_l, __uint_as_float(r[i + 1]) * inv_l);
          v.y = pack_bf16(__uint_as_float(r[i + 2]) * inv_l, __uint_as_float(r[i + 3]) * inv_l);
          v.z = pack_bf16(__uint_as_float(r[i + 4]) * inv_l, __uint_as_float(r[i + 5]) * inv_l);
          v.w = pack_bf16(__uint_as_float(r[i + 6]) * inv_l, __uint_as_float(r[i + 7]) * inv_l);
          *reinterpret_cast<uint4*>(orow + i) = v;
        }
      }
    }
    if (row < n_valid && w == 0) lse[(size_t)h * a.ld_lse + r0 + row] = (m_ref + __log2f(l)) * 0.6931471805599453f;
  }
  tc_fence_before();
  cluster_sync_all();                                   // no arrival or MMA still targets either CTA
  if (warp == kMma) tmem_dealloc_pair<512>(tmem);
}

}  // namespace fwd

static unsigned long long* fwd_trace_buffer() {
  static unsigned long long* buf = nullptr;
  static bool init = false;
  if (!init) {
    init = true;
    if (getenv("SKR_TRACE")) {
      cudaMalloc(&buf, 8192 * sizeof(unsigned long long));
      cudaMemset(buf, 0, 8192 * sizeof(unsigned long long));
      cudaMemcpyToSymbol(fwd::g_trace, &buf, sizeof(buf));
    }
  }
  return buf;
}

// Debug aid: copy the last fwd trace (event << 48 | clock) to host; returns the number of entries.
extern "C" __attribute__((visibility("default"))) int skr_debug_fwd_trace(unsigned long long* out, int cap) {
  unsigned long long* buf = fwd_trace_buffer();
  if (!buf) return 0;
  const int n = cap < 8192 ? cap : 8192;
  cudaMemcpy(out, buf, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaMemset(buf, 0, 8192 * sizeof(unsigned long long));
  return n;
}

// The CTA-pair d = 128 forward is a build-time variant (libskrull_fwd2sm.so, -DSKR_FWD_2SM_BUILD):
// skr_attn_block_m's answer is then fixed for the library, not switched by the environment.
bool fwd_two_sm() {
#ifdef SKR_FWD_2SM_BUILD
  return true;
#else
  return false;
#endif
}

skr_status sm100_attn_fwd(const AttnArgs& a, int d, const void* q, const void* k, const void* v, void* o, float* lse,
                          int n_q_rows, int n_kv_rows, cudaStream_t st) {
  fwd_trace_buffer();
  if (a.n_tiles == 0) return SKR_OK;
  CUtensorMap tq, tk, tv;
  const uint64_t qcols = (uint64_t)a.hq * d, kcols = (uint64_t)a.hkv * d;
  if (!make_tmap_2d(&tq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n_q_rows, qcols, qcols, fwd::BM, 64, true) ||
      !make_tmap_2d(&tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n_kv_rows, kcols, kcols,
                    d == 128 ? fwd::Cfg<128>::BN : fwd::Cfg<64>::BN, 64, true) ||
      !make_tmap_2d(&tv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n_kv_rows, kcols, kcols,
                    d == 128 ? fwd::Cfg<128>::BN : fwd::Cfg<64>::BN, 64, true))
    return fail(SKR_E_CUDA, "attn fwd: tensor map encode failed");
  // d = 128: consecutive q-head pairs over all heads (may straddle a GQA group, pairs_per_group = 0);
  // d = 64: pairs within each group
  const int ppg = d == 128 ? 0 : (a.hq / a.hkv + 1) / 2;
  const int n_pairs = d == 128 ? (a.hq + 1) / 2 : a.hkv * ppg;
  const int head_major = d == 128 ? 1 : 0;
  dim3 grid = head_major ? dim3(a.n_tiles, n_pairs) : dim3(n_pairs, a.n_tiles);
  // share of exponentials on the FMA pipe (MUFU ex2 bounds the d = 64 forward); SKR_FWD_POLY overrides
  static int poly = [] {
    const char* e = getenv("SKR_FWD_POLY");
    const int v = e ? atoi(e) : -1;
    return (v >= 0 && v <= 4) ? v : -1;
  }();
  // measured (profiles/fwd_period.py, S = 32K): d=64 best at 2/8, d=128 at 1/8; beyond that the
  // polynomial's FMA / ALU instructions cost more issue slots than the MUFU time they save
  const int pp = poly >= 0 ? poly : (d == 64 ? 2 : 1);
  auto launch = [&](auto kern, int smem, int threads = fwd::kThreads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<grid, threads, smem, st>>>(tq, tk, tv, a, (__nv_bfloat16*)o, lse, ppg, head_major);
  };
  // d = 128, one head per CTA (double-buffered S, separate P): opt-in, SKR_FWD_1H=1 (measured slower:
  // without the GQA head pair each K/V tile is loaded and read per head, profiles/r01_experiments.md)
  static int one_head = [] {
    const char* e = getenv("SKR_FWD_1H");
    return e ? atoi(e) : 0;
  }();
  // d = 128, one head per CTA PAIR (cta_group::2): opt-in, SKR_FWD_2SM=1
  if (d == 128 && fwd_two_sm()) {
    CUtensorMap tk2;   // K tiles are loaded in halves of 64 keys (one per CTA of the pair)
    if (!make_tmap_2d(&tk2, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n_kv_rows, kcols, kcols, 64, 64, true))
      return fail(SKR_E_CUDA, "attn fwd 2sm: tensor map encode failed");
    constexpr int smem = fwd::Cfg2sm::kSmem;
    dim3 g2(2 * a.hq, a.n_tiles);
    auto launch2 = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<g2, 320, smem, st>>>(tq, tk2, tv, a, (__nv_bfloat16*)o, lse);
    };
    if (pp == 0) launch2(fwd::attn_fwd2sm_kernel<0>);
    else if (pp == 1) launch2(fwd::attn_fwd2sm_kernel<1>);
    else launch2(fwd::attn_fwd2sm_kernel<2>);
    return launch_status("attn_fwd2sm_kernel");
  }
  if (d == 128 && one_head) {
    constexpr int smem = fwd::Cfg1h::kSmem;
    dim3 g1(a.hq, a.n_tiles);
    auto launch1 = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<g1, fwd::kThreads, smem, st>>>(tq, tk, tv, a, (__nv_bfloat16*)o, lse);
    };
    if (pp == 0) launch1(fwd::attn_fwd1h_kernel<0>);
    else if (pp == 1) launch1(fwd::attn_fwd1h_kernel<1>);
    else launch1(fwd::attn_fwd1h_kernel<2>);
    return launch_status("attn_fwd1h_kernel");
  }
  if (d == 128) {
    constexpr int smem = fwd::Cfg<128>::kSmem;
#if SKR_FWD_WG128 == 1
    constexpr int t1 = (8 * 1 + 2) * 32;   // one softmax warpgroup per head
    switch (pp) {
      case 0: launch(fwd::attn_fwd_kernel<128, 0, 1>, smem, t1); break;
      case 1: launch(fwd::attn_fwd_kernel<128, 1, 1>, smem, t1); break;
      default: launch(fwd::attn_fwd_kernel<128, 2, 1>, smem, t1); break;
    }
#else
    switch (pp) {
      case 0: launch(fwd::attn_fwd_kernel<128, 0>, smem); break;
      case 1: launch(fwd::attn_fwd_kernel<128, 1>, smem); break;
      case 2: launch(fwd::attn_fwd_kernel<128, 2>, smem); break;
      case 3: launch(fwd::attn_fwd_kernel<128, 3>, smem); break;
      default: launch(fwd::attn_fwd_kernel<128, 4>, smem); break;
    }
#endif
  } else if (d == 64) {
    constexpr int smem = fwd::Cfg<64>::kSmem;
#if SKR_FWD_WG64 == 1
    constexpr int t1 = (8 * 1 + 2) * 32;   // one softmax warpgroup per head
    switch (pp) {
      case 0: launch(fwd::attn_fwd_kernel<64, 0, 1>, smem, t1); break;
      case 1: launch(fwd::attn_fwd_kernel<64, 1, 1>, smem, t1); break;
      case 2: launch(fwd::attn_fwd_kernel<64, 2, 1>, smem, t1); break;
      default: launch(fwd::attn_fwd_kernel<64, 3, 1>, smem, t1); break;
    }
    return launch_status("attn_fwd_kernel");
#endif
    switch (pp) {
      case 0: launch(fwd::attn_fwd_kernel<64, 0>, smem); break;
      case 1: launch(fwd::attn_fwd_kernel<64, 1>, smem); break;
      case 2: launch(fwd::attn_fwd_kernel<64, 2>, smem); break;
      case 3: launch(fwd::attn_fwd_kernel<64, 3>, smem); break;
      default: launch(fwd::attn_fwd_kernel<64, 4>, smem); break;
    }
  } else {
    return fail(SKR_E_UNSUPPORTED, "bf16 attention supports d in {64, 128}");
  }
  return launch_status("attn_fwd_kernel");
}

}  // namespace skr
