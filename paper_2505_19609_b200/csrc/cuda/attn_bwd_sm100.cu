// Row a8: packed varlen causal attention backward on sm_100a (tcgen05 + TMEM + TMA).
//
// Plain definition (oracle/attention.py): P = exp(scale QK^T - LSE), dV = P^T dO,
// dP = dO V^T, D = rowsum(dO o O), dS = P o (dP - D), dQ = scale dS K, dK = scale dS^T Q;
// GQA sums dK/dV over the group's q-heads (R30).
//
// Work unit (CTA): one 128-key tile of one segment x one KV head g. It loops over the group's
// q-heads and the query tiles that can see the key tile (causal: query position >= key position),
// accumulating dK and dV in TMEM, so no cross-CTA reduction is needed for them.
//   d = 128: query step BQ = 64.  TMEM: S^T[0,64) dP^T[64,128) dQ^T[128,192) dV[256,384) dK[384,512)
//            dQ^T = K^T dS^T (M = d): thread = feature, reductions coalesced along d.
//   d =  64: query step BQ = 128. TMEM: S^T[0,128) dP^T[128,256) dQ[256,320) dV[320,384) dK[384,448)
//            dQ = dS K (M = query rows).
// Warp roles (448 threads): warps 0-7 two compute warpgroups (thread = key row; warpgroup w owns
// query columns [w*BQ/2, (w+1)*BQ/2): P^T, dS^T from TMEM -> bf16 swizzled smem), warps 8-11 dQ
// (TMEM -> scaled fp32 SW128 smem tile -> one TMA bulk reduce-add per 32-column box into the fp32
// dQ accumulator), warp 12 TMA producer (K, V once; Q/dO ring of 2 + LSE/D rows), warp 13 MMA.
// MMA order per step n: S(n+1) as soon as S(n) is read | dV(n) after P(n) | dP(n+1) as soon as dP(n)
// is read | dK(n) dQ(n) after dS(n): the tensor core runs ahead while the compute warpgroups work.
#include <cstdlib>

#include "attn_common.cuh"
#include "device.cuh"
#include "sm100.cuh"
#include "tma.h"

namespace skr {
namespace bwd {

// Debug timeline (SKR_TRACE=1): (event, clock) pairs of block (0, 0) into a device buffer.
__device__ unsigned long long* g_trace = nullptr;
__device__ int g_skip_math = 0;   // debug: compute / dQ warpgroups only signal (pipeline timing)
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
__device__ __forceinline__ void trace(int ev) {
#ifdef SKR_KERNEL_TRACE   // debug builds only: production kernels carry no instrumentation
  unsigned long long* buf = g_trace_smem;
  if (buf != nullptr) {
    const int role = ev / 10 < 8 ? ev / 10 : 7;
    const int i = g_trace_cnt[role]++;
    buf[role * 1024 + (i & 1023)] = ((unsigned long long)ev << 48) | (clock64() & 0xFFFFFFFFFFFFull);
  }
#endif
}

constexpr int BN = 128;  // key tile
// Grid order (launch argument head_major): 0 = (KV head, key tile) with the head fastest; 1 = (key
// tile, KV head), every key tile of one KV head before the next, so the CTAs in flight share one
// group's Q / dO / dQ rows. d = 128 uses 1 (S4n1 bwd DRAM 166 -> 120 GB per launch, C5n1 bwd
// -5 %); d = 64 keeps 0 (profiles/r02_experiments.md).
constexpr int kThreads = 448;
// scale * P folded into the exponent (see the producer warp): S4n1 backward -9 % instructions but
// only +0.3 % S4n1, and LESS accurate -- scale (1/sqrt(d), not a power of two) moves the large P
// values into the coarse start of their bf16 binade (P ~ 1 -> 0.088: relative ulp 2^-7.5 instead of
// 2^-8), which doubled the share of dV elements above 2e-2 and failed the C3n2 full-size parity
// (profiles/r02_experiments.md). Off: the exact arithmetic is the default.
#ifndef SKR_BWD_SCALE_FOLD
#define SKR_BWD_SCALE_FOLD 0
#endif
constexpr bool kFold = SKR_BWD_SCALE_FOLD;
constexpr int kComputeThreads = 256;

template <int D>
struct Cfg {
  static constexpr int BQ = D == 128 ? 64 : 128;         // query step
  static constexpr int H = BQ / 2;                       // columns per compute warpgroup
  static constexpr int kStages = 3;                      // Q/dO (+LSE/D) ring depth
  static constexpr int kChunks = D / 64;
  static constexpr int kKVBytes = BN * D * 2;
  static constexpr int kQBytes = BQ * D * 2;
  static constexpr int kPBytes = BN * BQ * 2;
  static constexpr int kDQBytes = BQ * D * 4;            // fp32 dQ tile, SW128 boxes of 32 columns
  static constexpr int kOffK = 0;
  static constexpr int kOffV = kOffK + kKVBytes;
  static constexpr int kOffQ = kOffV + kKVBytes;          // [kStages]
  static constexpr int kOffDO = kOffQ + kStages * kQBytes; // [kStages]
  static constexpr int kOffDS = kOffDO + kStages * kQBytes;
  static constexpr int kOffDQ = kOffDS + kPBytes;
  // d = 64: -LSE/scale and -D enter the S^T / dP^T accumulators through one K = 16 MMA each
  // (ones[128 x 16] x split[16 x BQ], the value as a 3-term bf16 split in k-rows 0-2), so the
  // compute warps never broadcast-load per-query values from shared memory (those loads were half
  // of all LSU shared traffic, profiles/r01_experiments.md). d = 128 keeps the smem rows.
  static constexpr bool kInit = D == 64;
  static constexpr int kInitBytes = 16 * BQ * 2;          // [16 k-rows][BQ] bf16, MN-major SW128 boxes
  static constexpr int kOnesBytes = 16 * BN * 2;          // [16 k-rows][BN] bf16 ones, MN-major
  static constexpr int kOffAux = kOffDQ + kDQBytes;       // kInit: [kStages][2] init tiles + ones;
                                                          // else lse2[kStages][BQ], dd[kStages][BQ] fp32
  static constexpr int kAuxBytes = kInit ? kStages * 2 * kInitBytes + kOnesBytes : 2 * kStages * BQ * 4;
  static constexpr int kOffBar = kOffAux + kAuxBytes;
  static constexpr int kSmem = kOffBar + 256 + 1024;
  // TMEM columns. P^T and dS^T (bf16 pairs) are the A operands of dV / dK straight from TMEM.
  //  d = 128: S^T[0,64) dP^T[64,128) dQ^T[128,192) P^T[192,224) dS^T[224,256) dV[256,384) dK[384,512)
  //  d =  64: S^T[0,128) dP^T[128,256) dQ[256,320) dV[320,384) dK[384,448) P^T[448,512);
  //           dS^T aliases dP^T: warpgroup w packs its 64 columns into [128+64w, 160+64w)
  //  d = 128 with kKT: K^T (bf16 pairs, lanes = features) is the TMEM A operand of dQ^T = K^T dS^T
  //           at [192,256), P^T / dS^T alias the warpgroup's own S^T / dP^T columns:
  //           S^T[0,64) (P^T at 32w) dP^T[64,128) (dS^T at 64+32w) dQ^T[128,192) K^T[192,256) dV dK
  static constexpr bool kDSAlias = D == 64;
#ifndef SKR_BWD_KT
#define SKR_BWD_KT 0   // measured slower (profiles/r01_experiments.md); kept as an option
#endif
  static constexpr bool kKT = D == 128 && SKR_BWD_KT;
  static constexpr int tS = 0;
  static constexpr int tDP = BQ;
  static constexpr int tDQ = 2 * BQ;
  static constexpr int tDV = D == 128 ? 256 : 320;
  static constexpr int tDK = 384;
  static constexpr int tPT = D == 128 ? 192 : 448;
  static constexpr int tKT = 192;
  // packed column of query pair-column q/2 for P^T / dS^T, per warpgroup half
  __device__ static constexpr int tDS(int w) {
    return kDSAlias ? 128 + 64 * w : (kKT ? BQ + H * w : 224 + (H / 2) * w);
  }
  __device__ static constexpr int tPTw(int w) { return kKT ? H * w : tPT + (H / 2) * w; }
};

struct Bars {
  uint64_t kv_full;
  uint64_t qdo_full[3], qdo_empty[3];
  uint64_t s_full, dp_full, p_full, ds_full, dv_done, dsq_done, dq_full, dq_empty;
  uint64_t s_free, dp_free;
  uint64_t mma_done;   // single phase: every MMA of the CTA has completed (dK / dV epilogue)
  uint64_t kt_full;    // kKT: K^T written to TMEM by the dQ warpgroup (128 arrivals)
  uint32_t tmem_base;
};

// Steps n = (q-head of the group, query tile); iterated incrementally by every role.
// SKR_BWD_ORDER 0: q-heads outer, query tiles ascending inner; 1: query tiles ascending outer, the
// group's q-heads inner (the CTAs in flight stay on nearby query rows for all heads); 2: query tiles
// DESCENDING outer, heads inner.
#ifndef SKR_BWD_ORDER
#define SKR_BWD_ORDER 0
#endif
struct StepIter {
  int hi, qt, qt_first, qt_last, grp;
  __device__ StepIter(int first, int last, int grp_)
      : hi(0), qt(SKR_BWD_ORDER == 2 ? last : first), qt_first(first), qt_last(last), grp(grp_) {}
  __device__ void next() {
    if (SKR_BWD_ORDER == 0) {
      if (++qt > qt_last) qt = qt_first, ++hi;
    } else if (++hi == grp) {
      hi = 0;
      qt += SKR_BWD_ORDER == 2 ? -1 : 1;
    }
  }
};

// kPolyPer8: how many of every 8 exponentials run as a polynomial on the FMA pipe (the exp phase of
// the two compute warpgroups is MUFU-bound).
template <int D, int kPolyPer8>
__global__ void __launch_bounds__(kThreads, 1)
    attn_bwd_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const __grid_constant__ CUtensorMap tm_do,
                    const __grid_constant__ CUtensorMap tm_dq, AttnArgs a, const float* __restrict__ lse,
                    const float* __restrict__ Dbuf, void* __restrict__ dk_out, void* __restrict__ dv_out,
                    int accumulate, float* __restrict__ dq_acc, float* __restrict__ dk_acc,
                    float* __restrict__ dv_acc, int head_major) {
  using C = Cfg<D>;
  constexpr int BQ = C::BQ, H = C::H;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  Bars* bars = reinterpret_cast<Bars*>(smem + C::kOffBar);
  float* aux = reinterpret_cast<float*>(smem + C::kOffAux);  // lse2[kStages][BQ] then dd[kStages][BQ]
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  const int g = head_major ? blockIdx.y : blockIdx.x;
  const int bt = head_major ? blockIdx.x : blockIdx.y;
  // work item {seg, key tile, q_lo, q_hi} (skr_tiles_bwd): the key tile against the segment-relative
  // queries [q_lo, q_hi) that see it; a band of a split tile (partial) adds its dK / dV in fp32
  const int32_t* item = a.tiles + 4 * bt;
  const int seg = item[0], ktile = item[1], q_lo = item[2], q_hi = item[3];
  const int grp = a.hq / a.hkv;
  const int cu0 = a.cu[seg], q_len = a.cu[seg + 1] - cu0;
  const int q_pos = a.q_pos[seg], k_len = a.k_len[seg], kst = a.k_start[seg];
  const int kv0 = ktile * BN;
  const int i_vis = max(0, kv0 - q_pos);            // first query (segment-relative) that sees the tile
  const bool partial = q_lo > i_vis || q_hi < q_len;
  const int i_first = max(i_vis, q_lo);             // band edges are multiples of 128, so of BQ
  const int qt_first = i_first / BQ, qt_last = (min(q_len, q_hi) - 1) / BQ;
  const int n_steps = grp * (qt_last - qt_first + 1);

  if (threadIdx.x == 0) {
    mbar_init(&bars->kv_full, 1);
    for (int s = 0; s < C::kStages; ++s) mbar_init(&bars->qdo_full[s], 33), mbar_init(&bars->qdo_empty[s], 1);
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->dp_full, 1);
    mbar_init(&bars->p_full, kComputeThreads);
    mbar_init(&bars->ds_full, kComputeThreads);
    mbar_init(&bars->dv_done, 1);
    mbar_init(&bars->dsq_done, 1);
    mbar_init(&bars->dq_full, 1);
    mbar_init(&bars->dq_empty, 128);
    mbar_init(&bars->s_free, kComputeThreads);
    mbar_init(&bars->dp_free, kComputeThreads);
    mbar_init(&bars->mma_done, 1);
    mbar_init(&bars->kt_full, 128);
    fence_mbar_init();
  }
  trace_init();
  if (C::kInit) {
    // zero the init tiles (k-rows 3-15 stay zero) and fill the ones tile, then hand them to the
    // async proxy (the MMA reads them)
    uint4* z = reinterpret_cast<uint4*>(smem + C::kOffAux);
    constexpr int nz = C::kStages * 2 * C::kInitBytes / 16, no = C::kOnesBytes / 16;
    for (int i = threadIdx.x; i < nz + no; i += kThreads)
      z[i] = i < nz ? make_uint4(0u, 0u, 0u, 0u) : make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    fence_async_smem();
  }
  if (warp == 13) tmem_alloc<512>(&bars->tmem_base);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 12) {
    // ================= TMA producer (+ LSE / D rows of each step into smem)
    if (elect_one()) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_do);
      tma_prefetch_desc(&tm_dq);
      mbar_expect_tx(&bars->kv_full, 2 * C::kKVBytes);
      for (int c = 0; c < C::kChunks; ++c) {
        tma_load_2d(smem + C::kOffK + c * BN * 128, &tm_k, &bars->kv_full, g * D + c * 64, kst + kv0);
        tma_load_2d(smem + C::kOffV + c * BN * 128, &tm_v, &bars->kv_full, g * D + c * 64, kst + kv0);
      }
    }
    // LSE / D of a step are fetched into registers one step ahead, so their global-load latency
    // overlaps the wait for the stage to free up instead of delaying the compute warpgroups.
    constexpr int kPer = BQ / 32;
    float pl[kPer], pd[kPer];
    const float inv_scale = 1.f / a.scale;
    // kFold: the compute warpgroups produce P' = scale * P (log2(scale) folded into the exponent's
    // bias: zero extra instructions), so dS' = scale * dS carries dQ's and dK's scale and the dQ
    // warpgroup stores the accumulator unscaled; dV' = scale * dV is divided once at the epilogue
    const float ln_scale = kFold ? logf(a.scale) : 0.f;
    auto fetch = [&](const StepIter& s_) {
      const int h = g * grp + s_.hi, q0 = s_.qt * BQ, nv = min(BQ, q_len - q0);
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int i = lane + 32 * u;
        const size_t off = (size_t)h * a.ld_lse + cu0 + q0 + i;
        if (C::kInit) {   // accumulator init values: S^T - LSE/scale, dP^T - D
          pl[u] = i < nv ? (ln_scale - lse[off]) * inv_scale : -1e30f;   // p = 0 for invalid queries
          pd[u] = i < nv ? -Dbuf[off] : 0.f;
        } else {
          pl[u] = i < nv ? (lse[off] - ln_scale) * 1.4426950408889634f : INFINITY;   // p = 0 for invalid queries
          pd[u] = i < nv ? Dbuf[off] : 0.f;
        }
      }
    };
    StepIter it(qt_first, qt_last, grp);
    fetch(it);
    for (int n = 0; n < n_steps; ++n) {
      const int st = n % C::kStages;
      const int h = g * grp + it.hi, q0 = it.qt * BQ;
      mbar_wait(&bars->qdo_empty[st], ((n / C::kStages) & 1) ^ 1);
      if (elect_one()) {
        mbar_expect_tx(&bars->qdo_full[st], 2 * C::kQBytes);
        for (int c = 0; c < C::kChunks; ++c) {
          tma_load_2d(smem + C::kOffQ + st * C::kQBytes + c * BQ * 128, &tm_q, &bars->qdo_full[st], h * D + c * 64,
                      cu0 + q0);
          tma_load_2d(smem + C::kOffDO + st * C::kQBytes + c * BQ * 128, &tm_do, &bars->qdo_full[st],
                      h * D + c * 64, cu0 + q0);
        }
      }
      if (C::kInit) {
        // 3-term bf16 split (hi + mid + lo carries ~24 bits) into k-rows 0-2 of column n
        const uint32_t tl = smem_u32(smem + C::kOffAux + (st * 2) * C::kInitBytes);
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          const int n = lane + 32 * u;
          const uint32_t col = (n / 64) * (16 * 128);
#pragma unroll
          for (int w = 0; w < 2; ++w) {
            float v = w == 0 ? pl[u] : pd[u];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
              const __nv_bfloat16 b = __float2bfloat16_rn(v);
              v -= __bfloat162float(b);
              st_shared_u16(tl + w * C::kInitBytes + col + sw128_off(k, n % 64), __bfloat16_as_ushort(b));
            }
          }
        }
        fence_async_smem();
      } else {
#pragma unroll
        for (int u = 0; u < kPer; ++u) {
          aux[st * BQ + lane + 32 * u] = pl[u];
          aux[C::kStages * BQ + st * BQ + lane + 32 * u] = pd[u];
        }
      }
      __syncwarp();
      mbar_arrive(&bars->qdo_full[st]);
      it.next();
      if (n + 1 < n_steps) fetch(it);
    }
  } else if (warp == 13) {
    // ================= MMA issuer (one elect.sync-elected thread; see below)
    const uint32_t sK = smem_u32(smem + C::kOffK), sV = smem_u32(smem + C::kOffV);
    const uint32_t sQ = smem_u32(smem + C::kOffQ), sDO = smem_u32(smem + C::kOffDO);
    const uint32_t sDS = smem_u32(smem + C::kOffDS);
    const uint32_t id_sdp = idesc_bf16_f32(BN, BQ, 0, 0);   // S^T = K Q^T, dP^T = V dO^T
    const uint32_t id_kv = idesc_bf16_f32(BN, D, 0, 1);     // dV += P^T dO, dK += dS^T Q
    // dQ^T = K^T dS^T (d = 128) or dQ = dS K (d = 64): both operands MN-major
    const uint32_t id_dq = D == 128 ? idesc_bf16_f32(D, BQ, 1, 1) : idesc_bf16_f32(BQ, D, 1, 1);
    // descriptor of (base + off) == descriptor of base + (off >> 4)
    const uint64_t dK = sdesc_sw128(sK, 16, 1024), dV = sdesc_sw128(sV, 16, 1024);
    const uint64_t dQ = sdesc_sw128(sQ, 16, 1024), dDO = sdesc_sw128(sDO, 16, 1024);
    const uint64_t dQmn = sdesc_sw128(sQ, BQ * 128, 1024), dDOmn = sdesc_sw128(sDO, BQ * 128, 1024);
    const uint64_t dKmn = sdesc_sw128(sK, BN * 128, 1024), dDSmn = sdesc_sw128(sDS, BN * 128, 1024);
    const uint64_t dK0 = sdesc_sw128(sK, 0, 1024), dDS0 = sdesc_sw128(sDS, 0, 1024);
    // kInit: ones[BN x 16] x init[16 x BQ] (both MN-major SW128, LBO = 64-column box stride) writes
    // -LSE/scale (S^T) or -D (dP^T) into every lane of the accumulator; the GEMM then accumulates
    const uint32_t id_init = idesc_bf16_f32(BN, BQ, 1, 1);
    const uint64_t dOnes = sdesc_sw128(smem_u32(smem + C::kOffAux + C::kStages * 2 * C::kInitBytes), 16 * 128, 1024);
    const uint64_t dInit = sdesc_sw128(smem_u32(smem + C::kOffAux), 16 * 128, 1024);
    auto issue_t = [&](uint64_t a_desc, uint64_t b_desc, uint32_t tcol, int init_tile) {
      if (C::kInit)
        umma_f16(tmem + tcol, dOnes, dInit + ((uint32_t)(init_tile * C::kInitBytes) >> 4), id_init, 0);
#pragma unroll
      for (int k = 0; k < D / 16; ++k) {
        const uint32_t ao = ((k / 4) * (BN * 128) + (k % 4) * 32) >> 4;
        const uint32_t bo = ((k / 4) * (BQ * 128) + (k % 4) * 32) >> 4;
        umma_f16(tmem + tcol, a_desc + ao, b_desc + bo, id_sdp, C::kInit || k > 0);
      }
    };
    // dV / dK: A = P^T or dS^T from TMEM (k-step = 16 queries = 8 packed columns of one warpgroup
    // half), B = dO or Q tile (MN-major over d)
    auto issue_kv = [&](bool is_dk, uint64_t b_desc, uint32_t tcol, bool acc) {
#pragma unroll
      for (int k = 0; k < BQ / 16; ++k) {
        const int w = (k * 16) / H, kk = (k * 16) % H;
        const uint32_t a_col = (is_dk ? C::tDS(w) : C::tPTw(w)) + kk / 2;
        umma_f16_ts(tmem + tcol, tmem + a_col, b_desc + ((uint32_t)(k * 2048) >> 4), id_kv, acc || k > 0);
      }
    };
    const uint32_t id_dq_ts = idesc_bf16_f32(D, BQ, 0, 1);   // kKT: A = K^T from TMEM, B = dS^T (MN-major)
    auto issue_dq = [&]() {
#pragma unroll
      for (int k = 0; k < BN / 16; ++k) {
        const uint32_t o = (uint32_t)(k * 2048) >> 4;
        if (C::kKT)
          umma_f16_ts(tmem + C::tDQ, tmem + C::tKT + k * 8, dDS0 + o, id_dq_ts, k > 0);
        else if (D == 128)
          umma_f16(tmem + C::tDQ, dKmn + o, dDS0 + o, id_dq, k > 0);
        else
          umma_f16(tmem + C::tDQ, dDSmn + o, dK0 + o, id_dq, k > 0);
      }
    };
    const uint32_t qstage = (uint32_t)C::kQBytes >> 4;
    // ONE elected thread runs the whole issue loop: re-entering an elected region per MMA group costs
    // ~200 cycles (descriptor R2UR + ELECT/BSSY) while the tensor pipe buffers only ~one MMA ahead of
    // the issuing thread (profiles/umma_probe.py), so per-group election left the pipe idle.
    if (elect_one()) {
      PhaseAcct pa;   // waits: 0 s_free, 1 qdo_full, 2 p_full, 3 dp_free, 4 ds_full, 5 dq_empty; 6 issue
      pa.start();
      mbar_wait_sleep(&bars->kv_full, 0);
      mbar_wait_sleep(&bars->qdo_full[0], 0);
      tc_fence_after();
      issue_t(dK, dQ, C::tS, 0);
      umma_commit(&bars->s_full);
      issue_t(dV, dDO, C::tDP, 1);
      umma_commit(&bars->dp_full);
      // kKT (d = 128): P^T / dS^T alias S^T / dP^T, so S(n+1) follows dV(n) and dP(n+1) follows dK(n)
      // in the in-order tensor pipe (p_full / ds_full also mean the compute warpgroups read S / dP).
      // Otherwise S(n+1) is issued as soon as the compute warpgroups have read S(n) out of TMEM (P^T
      // has its own columns); dP(n+1) likewise for d = 128, while for d = 64 (dS^T aliases dP^T) it
      // follows dK(n).
      for (int n = 0; C::kKT && n < n_steps; ++n) {
        const int st = n % C::kStages, st1 = (n + 1) % C::kStages;
        const bool more = n + 1 < n_steps;
        pa.mark(6);
        mbar_wait_sleep(&bars->p_full, n & 1);
        pa.mark(2);
        tc_fence_after();
        issue_kv(false, dDOmn + st * qstage, C::tDV, n > 0);
        umma_commit(&bars->dv_done);
        if (more) {
          pa.mark(6);
          mbar_wait_sleep(&bars->qdo_full[st1], ((n + 1) / C::kStages) & 1);
          pa.mark(1);
          tc_fence_after();
          issue_t(dK, dQ + st1 * qstage, C::tS, 2 * st1);
          umma_commit(&bars->s_full);
        }
        pa.mark(6);
        mbar_wait_sleep(&bars->ds_full, n & 1);
        pa.mark(4);
        tc_fence_after();
        issue_kv(true, dQmn + st * qstage, C::tDK, n > 0);
        if (more) {
          issue_t(dV, dDO + st1 * qstage, C::tDP, 2 * st1 + 1);
          umma_commit(&bars->dp_full);
        }
        pa.mark(6);
        if (n == 0) mbar_wait_sleep(&bars->kt_full, 0);
        mbar_wait_sleep(&bars->dq_empty, (n & 1) ^ 1);
        pa.mark(5);
        tc_fence_after();
        issue_dq();
        umma_commit(&bars->dq_full);
        umma_commit(&bars->dsq_done);
        umma_commit(&bars->qdo_empty[st]);
      }
      for (int n = 0; !C::kKT && n < n_steps; ++n) {
        const int st = n % C::kStages, st1 = (n + 1) % C::kStages;
        const bool more = n + 1 < n_steps;
        pa.mark(6);
        mbar_wait_sleep(&bars->s_free, n & 1);
        pa.mark(0);
        trace(1);
        if (more) {
          pa.mark(6);
          mbar_wait_sleep(&bars->qdo_full[st1], ((n + 1) / C::kStages) & 1);
          pa.mark(1);
          trace(2);
          tc_fence_after();
          issue_t(dK, dQ + st1 * qstage, C::tS, 2 * st1);
          umma_commit(&bars->s_full);
        }
        pa.mark(6);
        mbar_wait_sleep(&bars->p_full, n & 1);
        pa.mark(2);
        trace(3);
        tc_fence_after();
        issue_kv(false, dDOmn + st * qstage, C::tDV, n > 0);
        umma_commit(&bars->dv_done);
        if (!C::kDSAlias) {
          pa.mark(6);
          mbar_wait_sleep(&bars->dp_free, n & 1);
          pa.mark(3);
          if (more) {
            tc_fence_after();
            issue_t(dV, dDO + st1 * qstage, C::tDP, 2 * st1 + 1);
            umma_commit(&bars->dp_full);
          }
        }
        pa.mark(6);
        mbar_wait_sleep(&bars->ds_full, n & 1);
        pa.mark(4);
        trace(4);
        tc_fence_after();
        issue_kv(true, dQmn + st * qstage, C::tDK, n > 0);
        // d = 64 (dS^T aliases dP^T): dP(n+1) may follow dK(n), the last reader of dS^T(n) in TMEM
        // (dQ(n) reads dS from smem), so it goes into the pipe before dQ(n) and its dq_empty wait
        if (C::kDSAlias && more) {
          issue_t(dV, dDO + st1 * qstage, C::tDP, 2 * st1 + 1);
          umma_commit(&bars->dp_full);
        }
        pa.mark(6);
        mbar_wait_sleep(&bars->dq_empty, (n & 1) ^ 1);
        pa.mark(5);
        trace(5);
        tc_fence_after();
        issue_dq();
        umma_commit(&bars->dq_full);
        umma_commit(&bars->dsq_done);
        umma_commit(&bars->qdo_empty[st]);
      }
      umma_commit(&bars->mma_done);
      pa.mark(6);
      pa.flush(g_trace_smem, 13);
#ifdef SKR_PHASE_ACCT
      if (g_trace_smem != nullptr) g_trace_smem[13 * 8 + 7] = (unsigned long long)n_steps;
#endif
    }
    __syncwarp();
  } else if (warp < 8) {
    // ================= two compute warpgroups: thread = key row, warpgroup = half of the query columns
    const int j = (warp % 4) * 32 + lane;
    const int col0 = (warp / 4) * H;              // this warpgroup's first query column
    const int kvp = kv0 + j;                      // key position
    const uint32_t lane_base = (uint32_t)((warp % 4) * 32) << 16;
    const float sl2 = a.scale * 1.4426950408889634f;
    const uint32_t sDS = smem_u32(smem + C::kOffDS);
    const uint32_t sAux = smem_u32(aux);
    const int wg = warp / 4;
    StepIter it(qt_first, qt_last, grp);
    // 0 wait Q/dO + S, 1 load S, 2 exp + mask, 3 wait dV done, 4 store P^T, 5 wait dP, 6 dS math, 7 store dS
    PhaseAcct pa;
    pa.start();
    for (int n = 0; n < n_steps; ++n, it.next()) {
      const int st = n % C::kStages;
      const int qp_base = q_pos + it.qt * BQ + col0;        // position of this warpgroup's first query
      // warp-uniform: causal mask needed, or the tile holds keys past k_len (invisible: ring CP)
      const bool diag = kv0 + BN - 1 > qp_base || kv0 + BN > k_len;
      mbar_wait(&bars->qdo_full[st], (n / C::kStages) & 1);
      if (threadIdx.x == 0) trace(14);
      const uint32_t a_lse = sAux + (st * BQ + col0) * 4, a_dd = sAux + (C::kStages * BQ + st * BQ + col0) * 4;
      mbar_wait(&bars->s_full, n & 1);
      pa.mark(0);
      if (threadIdx.x == 0) trace(10);
      tc_fence_after();
      float p[H];
#pragma unroll
      for (int c = 0; c < H; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem + lane_base + C::tS + col0 + c, r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) p[c + i] = __uint_as_float(r[i]);
      }
      tc_fence_before();
      mbar_arrive(&bars->s_free);                   // S TMEM may be overwritten by S(n+1)
      pa.mark(1);
      const float2 sl2_2 = make_float2(sl2, sl2);
#pragma unroll
      for (int i = 0; i < H; i += 4) {
        float2 e0, e1;
        if (C::kInit) {   // the accumulator already holds s - LSE/scale
          e0 = fmul2(make_float2(p[i], p[i + 1]), sl2_2);
          e1 = fmul2(make_float2(p[i + 2], p[i + 3]), sl2_2);
        } else {
          const float4 l4 = ld_shared_f4(a_lse + i * 4);     // -lse2 is folded: p * sl2 - lse2
          e0 = ffma2(make_float2(p[i], p[i + 1]), sl2_2, make_float2(-l4.x, -l4.y));
          e1 = ffma2(make_float2(p[i + 2], p[i + 3]), sl2_2, make_float2(-l4.z, -l4.w));
        }
        // element (i % 8) < kPolyPer8 on the FMA pipe, the rest on MUFU
        p[i + 0] = (i % 8) + 0 < kPolyPer8 ? ex2_poly(e0.x) : ex2(e0.x);
        p[i + 1] = (i % 8) + 1 < kPolyPer8 ? ex2_poly(e0.y) : ex2(e0.y);
        p[i + 2] = (i % 8) + 2 < kPolyPer8 ? ex2_poly(e1.x) : ex2(e1.x);
        p[i + 3] = (i % 8) + 3 < kPolyPer8 ? ex2_poly(e1.y) : ex2(e1.y);
      }
      if (diag) {
#pragma unroll
        for (int i = 0; i < H; ++i)
          if (kvp > qp_base + i || kvp >= k_len) p[i] = 0.f;   // causal (invalid queries: lse2 = +inf -> 0)
      }
      pa.mark(2);
      if (n > 0) mbar_wait(&bars->dv_done, (n - 1) & 1);     // P^T TMEM columns free
      pa.mark(3);
      tc_fence_after();
      {
        uint32_t pk[H / 2];
#pragma unroll
        for (int i = 0; i < H / 2; ++i) pk[i] = pack_bf16(p[2 * i], p[2 * i + 1]);
        tmem_st_half<H / 2>(tmem + lane_base + C::tPTw(wg), pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars->p_full);
      if (threadIdx.x == 0) trace(11);
      pa.mark(4);
      mbar_wait(&bars->dp_full, n & 1);
      if (threadIdx.x == 0) trace(12);
      pa.mark(5);
      tc_fence_after();
      {
        // dP^T loads: all in flight under one wait where the registers allow (d = 128: 32 columns per
        // warpgroup); d = 64 holds 64 P values already, so one 32-column chunk at a time
        constexpr int kBatch = H <= 32 ? H / 32 : 1;
#pragma unroll
        for (int cb = 0; cb < H; cb += 32 * kBatch) {
          uint32_t r[kBatch][32];
#pragma unroll
          for (int b = 0; b < kBatch; ++b) tmem_ld32(tmem + lane_base + C::tDP + col0 + cb + 32 * b, r[b]);
          tmem_wait_ld();
          if (!C::kDSAlias && cb + 32 * kBatch >= H) {
            // dP TMEM may be overwritten by dP(n+1). (d = 64: dS^T aliases dP^T, so dP(n+1) is
            // ordered after this step's ds_full instead and dp_free is not used -- an arrive nobody
            // waits for is what compute-sanitizer's synccheck flagged)
            tc_fence_before();
            mbar_arrive(&bars->dp_free);
          }
#pragma unroll
          for (int b = 0; b < kBatch; ++b)
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              const int c = cb + 32 * b;
              float2 t0 = make_float2(__uint_as_float(r[b][i]), __uint_as_float(r[b][i + 1]));
              float2 t1 = make_float2(__uint_as_float(r[b][i + 2]), __uint_as_float(r[b][i + 3]));
              if (!C::kInit) {   // kInit: the accumulator already holds dP - D
                const float4 d4 = ld_shared_f4(a_dd + (c + i) * 4);
                t0 = fadd2(t0, make_float2(-d4.x, -d4.y));
                t1 = fadd2(t1, make_float2(-d4.z, -d4.w));
              }
              const float2 s0 = fmul2(make_float2(p[c + i], p[c + i + 1]), t0);
              const float2 s1 = fmul2(make_float2(p[c + i + 2], p[c + i + 3]), t1);
              p[c + i + 0] = s0.x, p[c + i + 1] = s0.y, p[c + i + 2] = s1.x, p[c + i + 3] = s1.y;
            }
        }
      }
      pa.mark(6);
      if (n > 0) mbar_wait(&bars->dsq_done, (n - 1) & 1);    // dS^T smem / TMEM free
      tc_fence_after();
      {
        uint32_t pk[H / 2];
#pragma unroll
        for (int i = 0; i < H / 2; ++i) pk[i] = pack_bf16(p[2 * i], p[2 * i + 1]);
        tmem_st_half<H / 2>(tmem + lane_base + C::tDS(wg), pk);   // A operand of dK
#pragma unroll
        for (int c = 0; c < H; c += 8) {                             // B (d = 128) / A (d = 64) of dQ
          const int cc = col0 + c;
          const uint32_t addr = sDS + (cc / 64) * (BN * 128) + sw128_off(j, cc % 64);
          st_shared_v4(addr, pk[c / 2], pk[c / 2 + 1], pk[c / 2 + 2], pk[c / 2 + 3]);
        }
      }
      tmem_wait_st();
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(&bars->ds_full);
      pa.mark(7);
      if (threadIdx.x == 0) trace(13);
    }
    if (lane == 0) pa.flush(g_trace_smem, warp);
    // ---- dK, dV epilogue: warpgroup 0 stores dK, warpgroup 1 stores dV
    mbar_wait(&bars->mma_done, 0);   // single-phase: no parity ambiguity however far a role ran ahead
    tc_fence_after();
    const bool valid = kvp < k_len;
    const size_t row = (size_t)(kst + kvp) * a.hkv + g;
    const int which = warp / 4;
    // accumulate == 2: this key row's partial goes to its owner's accumulator (peer memory);
    // accumulate == 0 and a band of a split tile: into the band accumulator (cast after the launch)
    float* const peer = (accumulate == 2 && valid) ? peer_row(a, which == 0, kst + kvp, g, D) : nullptr;
    float* const acc_f32 = accumulate == 2   ? peer
                           : accumulate == 1 ? reinterpret_cast<float*>(which == 0 ? dk_out : dv_out) + row * D
                           : partial         ? (which == 0 ? dk_acc : dv_acc) + row * D
                                             : nullptr;
    const uint32_t tcol = which == 0 ? C::tDK : C::tDV;
    const float mul = kFold ? (which == 0 ? 1.f : 1.f / a.scale) : (which == 0 ? a.scale : 1.f);
#pragma unroll
    for (int c = 0; c < D; c += 32) {
      uint32_t r[32];
      tmem_ld32(tmem + lane_base + tcol + c, r);
      tmem_wait_ld();
      if (!valid) continue;
      if (acc_f32 != nullptr) {
        float* dst = acc_f32 + c;
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          red_add_v4(dst + i, __uint_as_float(r[i]) * mul, __uint_as_float(r[i + 1]) * mul,
                     __uint_as_float(r[i + 2]) * mul, __uint_as_float(r[i + 3]) * mul);
      } else {
        __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(which == 0 ? dk_out : dv_out) + row * D + c;
#pragma unroll
        for (int i = 0; i < 32; i += 8) {
          uint4 v;
          v.x = pack_bf16(__uint_as_float(r[i]) * mul, __uint_as_float(r[i + 1]) * mul);
          v.y = pack_bf16(__uint_as_float(r[i + 2]) * mul, __uint_as_float(r[i + 3]) * mul);
          v.z = pack_bf16(__uint_as_float(r[i + 4]) * mul, __uint_as_float(r[i + 5]) * mul);
          v.w = pack_bf16(__uint_as_float(r[i + 6]) * mul, __uint_as_float(r[i + 7]) * mul);
          *reinterpret_cast<uint4*>(dst + i) = v;
        }
      }
    }
  } else {
    // ================= dQ warpgroup (warps 8-11): TMEM -> fp32 SW128 smem tile -> TMA reduce-add
    const int t = (warp - 8) * 32 + lane;         // TMEM lane
    const uint32_t lane_base = (uint32_t)((warp - 8) * 32) << 16;
    const uint32_t sDQ = smem_u32(smem + C::kOffDQ);
    constexpr int kBoxes = D / 32;                 // 32-column fp32 boxes
    constexpr int kBoxBytes = BQ * 128;
    if (C::kKT) {
      // K^T into TMEM (lane = feature t, packed key pairs): the A operand of every dQ^T MMA
      mbar_wait(&bars->kv_full, 0);
      const uint32_t kb = smem_u32(smem + C::kOffK) + (t / 64) * (BN * 128);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int key = 2 * (32 * c + i);
          const uint32_t lo = ld_shared_u16(kb + sw128_off(key, t % 64));
          const uint32_t hi = ld_shared_u16(kb + sw128_off(key + 1, t % 64));
          pk[i] = lo | (hi << 16);
        }
        tmem_st32(tmem + lane_base + C::tKT + 32 * c, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bars->kt_full);
    }
    // kFold: dS' already carries the scale (the multiply is a no-op the compiler drops)
    const float dq_mul = kFold ? 1.f : a.scale;
    StepIter it(qt_first, qt_last, grp);
    PhaseAcct pa;   // 0 wait dQ, 1 wait smem tile free, 2 TMEM -> smem, 3 issue reduce
    pa.start();
    for (int n = 0; n < n_steps; ++n, it.next()) {
      const int h = g * grp + it.hi, q0 = it.qt * BQ;
      mbar_wait(&bars->dq_full, n & 1);
      pa.mark(0);
      if (t == 0) trace(20);
      tc_fence_after();
      if (D == 128) {
        // dQ^T: lane = feature t, columns = queries of the step. Staged as two 16 KB halves (queries
        // [0,32) and [32,64)), each four SW128 boxes [32 q][32 f], double-buffered so the stores of
        // one half overlap the TMA reduce of the other (and of the previous step): the dQ
        // warpgroup's store -> reduce -> tile-free chain was the d = 128 critical path
        // (profiles/r01_experiments.md). Element (q, t) of a box sits at q * 128 + (((t / 4) ^
        // (q % 8)) * 16) + (t % 4) * 4: eight per-thread offsets (q % 8) plus q * 128 immediates.
        uint32_t r[BQ / 32][32];
#pragma unroll
        for (int c = 0; c < BQ; c += 32) tmem_ld32(tmem + lane_base + C::tDQ + c, r[c / 32]);
        tmem_wait_ld();
        tc_fence_before();
        mbar_arrive(&bars->dq_empty);              // the step's dQ^T is in registers
        pa.mark(1);
        constexpr int kHalfBytes = 32 * D * 4, kHBox = 32 * 128;
#pragma unroll
        for (int hh = 0; hh < BQ / 32; ++hh) {
          // the reduce that last read this half (two bulk groups ago) must be done
          if (warp == 8 && elect_one()) bulk_wait_read<1>();
          named_bar_sync(1, 128);
          const uint32_t hb = sDQ + hh * kHalfBytes + (t / 32) * kHBox + (t & 3) * 4;
          uint32_t off[8];
#pragma unroll
          for (int m = 0; m < 8; ++m) off[m] = hb + ((((t % 32) >> 2) ^ m) << 4);
#pragma unroll
          for (int q = 0; q < 32; ++q) st_shared_f32(off[q % 8] + q * 128, __uint_as_float(r[hh][q]) * dq_mul);
          fence_async_smem();
          named_bar_sync(1, 128);
          if (warp == 8) {
            if (elect_one()) {
              if (q0 + 32 * hh < q_len) {            // rows past the segment would only add zeros
#pragma unroll
                for (int b = 0; b < D / 32; ++b)
                  tma_reduce_add_2d(&tm_dq, smem + C::kOffDQ + hh * kHalfBytes + b * kHBox, h * D + b * 32,
                                    cu0 + q0 + 32 * hh);
              }
              bulk_commit();                           // one group per half, empty or not
            }
            __syncwarp();
          }
        }
        pa.mark(2);
      } else {
        // the previous step's reduce must have finished reading the smem tile
        if (warp == 8 && elect_one()) bulk_wait_read<0>();
        named_bar_sync(1, 128);
        pa.mark(1);
        // dQ: lane = query row t, columns = features
#pragma unroll
        for (int c = 0; c < D; c += 32) {
          uint32_t r[32];
          tmem_ld32(tmem + lane_base + C::tDQ + c, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            st_shared_f4(sDQ + (c / 32) * kBoxBytes + sw128_off_f32(t, i), __uint_as_float(r[i]) * dq_mul,
                         __uint_as_float(r[i + 1]) * dq_mul, __uint_as_float(r[i + 2]) * dq_mul,
                         __uint_as_float(r[i + 3]) * dq_mul);
        }
        tc_fence_before();
        mbar_arrive(&bars->dq_empty);                // TMEM dQ columns may be overwritten
        pa.mark(2);
        if (t == 0) trace(21);
        fence_async_smem();
        named_bar_sync(1, 128);
        if (warp == 8) {
          if (elect_one()) {
#pragma unroll
            for (int b = 0; b < kBoxes; ++b)
              tma_reduce_add_2d(&tm_dq, smem + C::kOffDQ + b * kBoxBytes, h * D + b * 32, cu0 + q0);
            bulk_commit();
          }
          __syncwarp();
        }
      }
      pa.mark(3);
    }
    if (lane == 0) pa.flush(g_trace_smem, warp);
    if (warp == 8 && elect_one()) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) tmem_dealloc<512>(tmem);
}

// D[h][r] = sum_c dO[r][h][c] * O[r][h][c] (bf16 in, fp32 out). A group of D/8 threads owns one
// (row, head): 16-byte loads of O and dO, shuffle-reduced inside the group. (The dQ accumulator is
// zeroed by a memset, which runs at copy bandwidth.)
template <int D>
__global__ void preprocess_kernel(int row_begin, int row_end, int hq, const __nv_bfloat16* __restrict__ o,
                                  const __nv_bfloat16* __restrict__ dout, float* __restrict__ Dbuf, int ld) {
  constexpr int G = D / 8;                       // threads per (row, head): 8 or 16
  const int64_t gid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G;
  const int sub = threadIdx.x % G;
  const int64_t row = row_begin + gid / hq;
  const int h = gid % hq;
  const bool ok = row < row_end;
  float s = 0.f;
  if (ok) {
    const size_t base = ((size_t)row * hq + h) * D + sub * 8;
    const uint4 a = *reinterpret_cast<const uint4*>(o + base);
    const uint4 b = *reinterpret_cast<const uint4*>(dout + base);
    const __nv_bfloat162* pa = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* pb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 x = __bfloat1622float2(pa[i]), y = __bfloat1622float2(pb[i]);
      s = fmaf(x.x, y.x, fmaf(x.y, y.y, s));
    }
  }
#pragma unroll
  for (int off = G / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (ok && sub == 0) Dbuf[(size_t)h * ld + row] = s;
}

__global__ void convert_dq_kernel(const float4* __restrict__ acc, uint2* __restrict__ dq, int64_t begin4,
                                  int64_t end4) {
  for (int64_t i = begin4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < end4;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = acc[i];
    uint2 o;
    o.x = pack_bf16(v.x, v.y);
    o.y = pack_bf16(v.z, v.w);
    dq[i] = o;
  }
}

}  // namespace bwd

static unsigned long long* trace_buffer() {
  static unsigned long long* buf = nullptr;
  static bool init = false;
  if (!init) {
    init = true;
    if (getenv("SKR_TRACE")) {
      cudaMalloc(&buf, 8192 * sizeof(unsigned long long));
      cudaMemset(buf, 0, 8192 * sizeof(unsigned long long));
      cudaMemcpyToSymbol(bwd::g_trace, &buf, sizeof(buf));
      const int skip = getenv("SKR_SKIP_MATH") ? 1 : 0;
      cudaMemcpyToSymbol(bwd::g_skip_math, &skip, sizeof(skip));
    }
  }
  return buf;
}

// Debug aid: copy the last bwd trace (event << 48 | clock) to host; returns the number of entries.
extern "C" __attribute__((visibility("default"))) int skr_debug_bwd_trace(unsigned long long* out, int cap) {
  unsigned long long* buf = trace_buffer();
  if (!buf) return 0;
  const int n = cap < 8192 ? cap : 8192;
  cudaMemcpy(out, buf, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  cudaMemset(buf, 0, 8192 * sizeof(unsigned long long));
  return n;
}

skr_status sm100_attn_bwd(const AttnArgs& a, int d, int row_begin, int row_end, const void* q, const void* k,
                          const void* v, const void* o, const void* dout, const float* lse, void* dq, void* dk,
                          void* dv, int accumulate, int dq_accumulate, float* Dbuf, float* dq_acc, float* dk_acc,
                          float* dv_acc, int n_q_rows, int n_kv_rows, cudaStream_t st) {
  // dq_accumulate (ring CP): dq is the caller's fp32 accumulator -- the kernel reduce-adds into it
  // directly, no zeroing and no bf16 conversion here
  if (dq_accumulate) dq_acc = static_cast<float*>(dq);
  trace_buffer();
  if (d != 64 && d != 128) return fail(SKR_E_UNSUPPORTED, "bf16 backward supports d in {64,128}");
  const int rows = row_end - row_begin;
  if (rows > 0) {
    const int64_t threads = (int64_t)rows * a.hq * (d / 8);
    const int blocks = (int)((threads + 255) / 256);
    if (d == 128)
      bwd::preprocess_kernel<128><<<blocks, 256, 0, st>>>(row_begin, row_end, a.hq, (const __nv_bfloat16*)o,
                                                          (const __nv_bfloat16*)dout, Dbuf, a.ld_lse);
    else
      bwd::preprocess_kernel<64><<<blocks, 256, 0, st>>>(row_begin, row_end, a.hq, (const __nv_bfloat16*)o,
                                                         (const __nv_bfloat16*)dout, Dbuf, a.ld_lse);
    if (skr_status e = launch_status("attn bwd preprocess")) return e;
    if (!dq_accumulate &&
        cudaMemsetAsync(dq_acc + (size_t)row_begin * a.hq * d, 0, (size_t)rows * a.hq * d * 4, st) != cudaSuccess)
      return fail(SKR_E_CUDA, "attn bwd: dQ accumulator memset");
  }
  if (a.n_tiles > 0) {
    CUtensorMap tq, tk, tv, tdo, tdq;
    const uint64_t qcols = (uint64_t)a.hq * d, kcols = (uint64_t)a.hkv * d;
    const uint32_t bq = d == 128 ? 64 : 128;
    if (!make_tmap_2d(&tq, q, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n_q_rows, qcols, qcols, bq, 64, true) ||
        !make_tmap_2d(&tdo, dout, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n_q_rows, qcols, qcols, bq, 64, true) ||
        !make_tmap_2d(&tk, k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n_kv_rows, kcols, kcols, bwd::BN, 64, true) ||
        !make_tmap_2d(&tv, v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n_kv_rows, kcols, kcols, bwd::BN, 64, true) ||
        !make_tmap_2d(&tdq, dq_acc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, n_q_rows, qcols, qcols,
                      d == 128 ? 32 : bq, 32, true))   // d = 128 reduces in 32-query halves
      return fail(SKR_E_CUDA, "attn bwd: tensor map encode failed");
    const int head_major = d == 128 ? 1 : 0;
    dim3 grid = head_major ? dim3(a.n_tiles, a.hkv) : dim3(a.hkv, a.n_tiles);
    // share of exponentials on the FMA pipe; SKR_BWD_POLY (0-3) overrides for sweeps
    static int poly = [] {
      const char* e = getenv("SKR_BWD_POLY");
      const int v = e ? atoi(e) : -1;
      return (v >= 0 && v <= 4) ? v : -1;
    }();
    // measured (C2 / C5n1 bench sweeps): d=64 best at 1/8 once the LSE/D loads left the exp phase
    // (it is then MUFU-bound), a loss at d=128 -> MUFU only
    const int pp = poly >= 0 ? poly : (d == 64 ? 1 : 0);
    auto launch = [&](auto kern, int smem) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      kern<<<grid, bwd::kThreads, smem, st>>>(tq, tk, tv, tdo, tdq, a, lse, Dbuf, dk, dv, accumulate, dq_acc,
                                              dk_acc, dv_acc, head_major);
    };
    if (d == 128) {
      constexpr int smem = bwd::Cfg<128>::kSmem;
      if (pp == 0) launch(bwd::attn_bwd_kernel<128, 0>, smem);
      else if (pp == 1) launch(bwd::attn_bwd_kernel<128, 1>, smem);
      else if (pp == 2) launch(bwd::attn_bwd_kernel<128, 2>, smem);
      else if (pp == 3) launch(bwd::attn_bwd_kernel<128, 3>, smem);
      else launch(bwd::attn_bwd_kernel<128, 4>, smem);
    } else {
      constexpr int smem = bwd::Cfg<64>::kSmem;
      if (pp == 0) launch(bwd::attn_bwd_kernel<64, 0>, smem);
      else if (pp == 1) launch(bwd::attn_bwd_kernel<64, 1>, smem);
      else if (pp == 2) launch(bwd::attn_bwd_kernel<64, 2>, smem);
      else if (pp == 3) launch(bwd::attn_bwd_kernel<64, 3>, smem);
      else launch(bwd::attn_bwd_kernel<64, 4>, smem);
    }
    if (skr_status e = launch_status("attn_bwd_kernel")) return e;
  }
  if (rows > 0 && !dq_accumulate) {
    const int64_t b4 = (int64_t)row_begin * a.hq * d / 4, e4 = (int64_t)row_end * a.hq * d / 4;
    const int blocks = (int)std::min<int64_t>((e4 - b4 + 255) / 256, 148 * 16);
    bwd::convert_dq_kernel<<<blocks, 256, 0, st>>>((const float4*)dq_acc, (uint2*)dq, b4, e4);
    if (skr_status e = launch_status("attn bwd dq convert")) return e;
  }
  return SKR_OK;
}

}  // namespace skr
