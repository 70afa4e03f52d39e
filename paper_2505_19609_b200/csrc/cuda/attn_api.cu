// C-ABI entry points of the attention kernels (rows a7/a8): argument checks and dispatch.
#include <algorithm>

#include "attn_common.cuh"
#include "device.cuh"
#include "sm100.cuh"

namespace skr {
bool fwd_two_sm();   // attn_fwd_sm100.cu: d = 128 forward on CTA pairs (the libskrull_fwd2sm.so build variant)
skr_status sm100_attn_fwd(const AttnArgs& a, int d, const void* q, const void* k, const void* v, void* o, float* lse,
                          int n_q_rows, int n_kv_rows, cudaStream_t st);
skr_status sm100_attn_bwd(const AttnArgs& a, int d, int row_begin, int row_end, const void* q, const void* k,
                          const void* v, const void* o, const void* dout, const float* lse, void* dq, void* dk,
                          void* dv, int accumulate, int dq_accumulate, float* Dbuf, float* dq_acc, float* dk_acc,
                          float* dv_acc, int n_q_rows, int n_kv_rows, cudaStream_t st);

// Query-banded backward work items (skr_tiles_bwd): the bands of one key tile each add an fp32
// partial dK / dV into an accumulator (ws) -- zeroed before the backward kernel and cast into dk / dv
// after it by the item of the tile's first band. One CTA per work item: the others exit at once, the
// owner zeroes / casts its key tile's rows for every KV head ([rows][hkv][d] is contiguous).
__global__ void __launch_bounds__(256) band_kv_kernel(AttnArgs a, int bn, int d, int convert,
                                                      float* __restrict__ dk_acc, float* __restrict__ dv_acc,
                                                      void* __restrict__ dk, void* __restrict__ dv, int out_bf16) {
  const int32_t* t = a.tiles + 4 * blockIdx.x;
  const int seg = t[0], kv0 = t[1] * bn, q_lo = t[2], q_hi = t[3];
  const int first_q = max(0, kv0 - a.q_pos[seg]);
  const bool partial = q_lo > first_q || q_hi < a.cu[seg + 1] - a.cu[seg];
  if (!partial || q_lo > first_q) return;                     // not split, or not the first band
  const int64_t r0 = a.k_start[seg] + kv0, r1 = a.k_start[seg] + min(kv0 + bn, a.k_len[seg]);
  const int64_t e0 = r0 * a.hkv * d / 4, e1 = r1 * a.hkv * d / 4;   // float4 index range
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    if (!convert) {
      reinterpret_cast<float4*>(dk_acc)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
      reinterpret_cast<float4*>(dv_acc)[e] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else if (out_bf16) {
      const float4 x = reinterpret_cast<const float4*>(dk_acc)[e], y = reinterpret_cast<const float4*>(dv_acc)[e];
      reinterpret_cast<uint2*>(dk)[e] = make_uint2(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w));
      reinterpret_cast<uint2*>(dv)[e] = make_uint2(pack_bf16(y.x, y.y), pack_bf16(y.z, y.w));
    } else {
      reinterpret_cast<float4*>(dk)[e] = reinterpret_cast<const float4*>(dk_acc)[e];
      reinterpret_cast<float4*>(dv)[e] = reinterpret_cast<const float4*>(dv_acc)[e];
    }
  }
}

// Ring CP (row f4): merge one partial attention result (O_p normalised, LSE_p natural log) into
// the running one (O_a fp32, LSE_a): L = log(e^LSE_a + e^LSE_p), O_a <- O_a e^(LSE_a - L) + O_p
// e^(LSE_p - L), LSE_a <- L -- the plain identity softmax over a union of disjoint key sets obeys.
// LSE = -inf marks an empty partial (weight 0). One warp per (row, head): the lanes read LSE_a before
// lane 0 overwrites it.
template <typename T>
__global__ void __launch_bounds__(256) merge_kernel(const T* __restrict__ o_p, const float* __restrict__ lse_p,
                                                    float* __restrict__ o_a, float* __restrict__ lse_a, int row_begin,
                                                    int row_end, int hq, int d, int ld, int first) {
  const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (w >= (int64_t)(row_end - row_begin) * hq) return;
  const int row = row_begin + (int)(w / hq), h = (int)(w % hq);
  const size_t lo = (size_t)h * ld + row, base = ((size_t)row * hq + h) * d;
  const float lp = lse_p[lo];
  float wa = 0.f, wp = 1.f, L = lp;
  if (!first) {
    const float la = lse_a[lo];
    const float mx = fmaxf(la, lp);
    if (mx == -INFINITY) return;                          // both empty: O_a stays 0, LSE_a -inf
    wa = expf(la - mx), wp = expf(lp - mx);
    const float den = wa + wp;                            // >= 1
    wa /= den, wp /= den;
    L = mx + logf(den);
  }
  for (int c = lane; c < d; c += 32) {
    const float x = (float)o_p[base + c];
    o_a[base + c] = first ? x : o_a[base + c] * wa + x * wp;
  }
  __syncwarp();
  if (lane == 0) lse_a[lo] = L;
}

static skr_status band_kv(const AttnArgs& a, int bn, int d, int convert, float* dk_acc, float* dv_acc, void* dk,
                          void* dv, int out_bf16, cudaStream_t st) {
  if (a.n_tiles == 0) return SKR_OK;
  band_kv_kernel<<<a.n_tiles, 256, 0, st>>>(a, bn, d, convert, dk_acc, dv_acc, dk, dv, out_bf16);
  return launch_status(convert ? "bwd band dK/dV cast" : "bwd band dK/dV zero");
}

static skr_status check_shape(const skr_attn_shape* s) {
  if (!s) return fail(SKR_E_ARG, "null shape");
  if (s->hq < 1 || s->hkv < 1 || s->hq % s->hkv) return fail(SKR_E_ARG, "hq must be a multiple of hkv");
  if (s->dtype == SKR_BF16) {
    if (s->d != 64 && s->d != 128) return fail(SKR_E_UNSUPPORTED, "bf16 kernels support d in {64,128}");
  } else if (s->dtype == SKR_FP32) {
    if (s->d != 32 && s->d != 64 && s->d != 128) return fail(SKR_E_UNSUPPORTED, "fp32 mode supports d in {32,64,128}");
  } else {
    return fail(SKR_E_ARG, "unknown dtype %d", s->dtype);
  }
  return SKR_OK;
}

static AttnArgs make_args(const skr_attn_shape* s, const skr_segs* g, int ld_lse) {
  AttnArgs a;
  a.cu = g->cu_seqlens_q;
  a.q_pos = g->q_pos;
  a.k_start = g->k_start;
  a.k_len = g->k_len;
  a.tiles = g->tiles;
  a.n_seg = g->n_seg;
  a.n_tiles = g->n_tiles;
  a.hq = s->hq;
  a.hkv = s->hkv;
  a.scale = s->scale;
  a.ld_lse = ld_lse;
  return a;
}

}  // namespace skr

using namespace skr;

SKR_EXPORT int32_t skr_attn_block_m(const skr_attn_shape* s) {
  if (s && s->dtype == SKR_FP32) return 32;
  return (s && s->d == 128 && fwd_two_sm()) ? 256 : 128;   // a CTA pair takes 256 query rows
}
SKR_EXPORT int32_t skr_attn_block_n(const skr_attn_shape* s) { return (s && s->dtype == SKR_FP32) ? 32 : 128; }

// Query-band height of the backward work items (skr_tiles_bwd). d = 128: a band's Q / dO / dQ rows
// for one KV group stay L2-resident while every key tile that sees them passes.
SKR_EXPORT int32_t skr_attn_bwd_band_rows(const skr_attn_shape* s) {
  return (s && s->dtype == SKR_BF16 && s->d == 128) ? 8192 : 0;
}

// ws layout: D [hq][n_q_rows] fp32 | bf16 only: dQ accumulator [n_q_rows][hq][d] fp32 | dK, dV band
// accumulators [n_q_rows][hkv][d] fp32 each (indexed by key row; kv_accumulate = 0 needs
// n_kv_rows <= n_q_rows)
static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
static size_t ws_dq_off(const skr_attn_shape* s, int32_t n) { return align256((size_t)s->hq * n * 4); }
static size_t ws_kv_off(const skr_attn_shape* s, int32_t n) {
  return ws_dq_off(s, n) + (s->dtype == SKR_FP32 ? 0 : align256((size_t)n * s->hq * s->d * 4));
}
static size_t ws_kv_bytes(const skr_attn_shape* s, int32_t n) { return align256((size_t)n * s->hkv * s->d * 4); }

SKR_EXPORT size_t skr_attn_bwd_ws_bytes(const skr_attn_shape* s, int32_t n_q_rows) {
  if (!s || n_q_rows < 0) return 0;
  return ws_kv_off(s, n_q_rows) + 2 * ws_kv_bytes(s, n_q_rows);
}

SKR_EXPORT skr_status skr_attn_merge(const skr_attn_shape* s, const void* o_part, const float* lse_part, float* o_acc,
                                     float* lse_acc, int32_t row_begin, int32_t row_end, int32_t ld_lse, int32_t first,
                                     void* stream) {
  if (skr_status e = check_shape(s)) return e;
  SKR_REQUIRE(row_begin >= 0 && row_begin <= row_end && row_end <= ld_lse, "skr_attn_merge: rows [%d,%d) / ld %d",
              row_begin, row_end, ld_lse);
  if (row_end == row_begin) return SKR_OK;
  SKR_REQUIRE(o_part && lse_part && o_acc && lse_acc, "skr_attn_merge: null pointer");
  if (skr_status e = check_sm100()) return e;
  const int64_t warps = (int64_t)(row_end - row_begin) * s->hq;
  const int blocks = (int)((warps * 32 + 255) / 256);
  cudaStream_t st = (cudaStream_t)stream;
  if (s->dtype == SKR_BF16)
    merge_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>((const __nv_bfloat16*)o_part, lse_part, o_acc, lse_acc,
                                                        row_begin, row_end, s->hq, s->d, ld_lse, first);
  else
    merge_kernel<float><<<blocks, 256, 0, st>>>((const float*)o_part, lse_part, o_acc, lse_acc, row_begin, row_end,
                                                s->hq, s->d, ld_lse, first);
  return launch_status("attn merge");
}

SKR_EXPORT skr_status skr_attn_fwd(const skr_attn_shape* s, const skr_segs* g, const void* q, const void* k,
                                   const void* v, void* o, float* lse, int32_t n_q_rows, int32_t n_kv_rows,
                                   void* stream) {
  if (skr_status e = check_shape(s)) return e;
  SKR_REQUIRE(g && n_q_rows >= 0 && n_kv_rows >= 0, "skr_attn_fwd: bad segments / sizes");
  if (g->n_tiles == 0) return SKR_OK;
  SKR_REQUIRE(q && k && v && o && lse && g->cu_seqlens_q && g->q_pos && g->k_start && g->k_len && g->tiles,
              "skr_attn_fwd: null pointer");
  if (skr_status e = check_sm100()) return e;
  AttnArgs a = make_args(s, g, n_q_rows);
  cudaStream_t st = (cudaStream_t)stream;
  if (s->dtype == SKR_FP32)
    return simt_attn_fwd(a, s->d, (const float*)q, (const float*)k, (const float*)v, (float*)o, lse, st);
  return sm100_attn_fwd(a, s->d, q, k, v, o, lse, n_q_rows, n_kv_rows, st);
}

static skr_status attn_bwd_impl(const skr_attn_shape* s, const skr_segs* g, const void* q, const void* k,
                                const void* v, const void* o, const void* dout, const float* lse, void* dq, void* dk,
                                void* dv, int32_t kv_accumulate, int32_t n_q_rows, int32_t n_kv_rows, void* ws,
                                size_t ws_bytes, void* stream, const uint64_t* peer_dk, const uint64_t* peer_dv,
                                const int32_t* row_map, int32_t pad_P, int32_t dq_accumulate = 0);

SKR_EXPORT skr_status skr_attn_bwd(const skr_attn_shape* s, const skr_segs* g, const void* q, const void* k,
                                   const void* v, const void* o, const void* dout, const float* lse, void* dq,
                                   void* dk, void* dv, int32_t kv_accumulate, int32_t n_q_rows, int32_t n_kv_rows,
                                   void* ws, size_t ws_bytes, void* stream) {
  SKR_REQUIRE(kv_accumulate == 0 || kv_accumulate == 1, "skr_attn_bwd: kv_accumulate must be 0 or 1");
  return attn_bwd_impl(s, g, q, k, v, o, dout, lse, dq, dk, dv, kv_accumulate, n_q_rows, n_kv_rows, ws, ws_bytes,
                       stream, nullptr, nullptr, nullptr, 0);
}

// Ring CP (row f4): every gradient is an fp32 accumulator the caller owns and zeroes; the call adds
// this segment class's contribution (dq [n_q_rows][hq][d], dk / dv [n_kv_rows][hkv][d], all fp32).
SKR_EXPORT skr_status skr_attn_bwd_acc(const skr_attn_shape* s, const skr_segs* g, const void* q, const void* k,
                                       const void* v, const void* o, const void* dout, const float* lse, float* dq,
                                       float* dk, float* dv, int32_t n_q_rows, int32_t n_kv_rows, void* ws,
                                       size_t ws_bytes, void* stream) {
  return attn_bwd_impl(s, g, q, k, v, o, dout, lse, dq, dk, dv, 1, n_q_rows, n_kv_rows, ws, ws_bytes, stream, nullptr,
                       nullptr, nullptr, 0, 1);
}

SKR_EXPORT skr_status skr_attn_bwd_peer(const skr_attn_shape* s, const skr_segs* g, const void* q, const void* k,
                                        const void* v, const void* o, const void* dout, const float* lse, void* dq,
                                        const uint64_t* peer_dk, const uint64_t* peer_dv, const int32_t* row_map,
                                        int32_t pad_rows_P, int32_t n_q_rows, int32_t n_kv_rows, void* ws,
                                        size_t ws_bytes, void* stream) {
  SKR_REQUIRE(peer_dk && peer_dv && row_map && pad_rows_P > 0, "skr_attn_bwd_peer: null peer table / P = 0");
  // dk / dv are unused in this mode; pass the peer tables so the null checks hold
  return attn_bwd_impl(s, g, q, k, v, o, dout, lse, dq, (void*)peer_dk, (void*)peer_dv, 2, n_q_rows, n_kv_rows, ws,
                       ws_bytes, stream, peer_dk, peer_dv, row_map, pad_rows_P);
}

static skr_status attn_bwd_impl(const skr_attn_shape* s, const skr_segs* g, const void* q, const void* k,
                                const void* v, const void* o, const void* dout, const float* lse, void* dq, void* dk,
                                void* dv, int32_t kv_accumulate, int32_t n_q_rows, int32_t n_kv_rows, void* ws,
                                size_t ws_bytes, void* stream, const uint64_t* peer_dk, const uint64_t* peer_dv,
                                const int32_t* row_map, int32_t pad_P, int32_t dq_accumulate) {
  if (skr_status e = check_shape(s)) return e;
  SKR_REQUIRE(g && n_q_rows >= 0 && n_kv_rows >= 0, "skr_attn_bwd: bad segments / sizes");
  SKR_REQUIRE(g->row_begin >= 0 && g->row_begin <= g->row_end && g->row_end <= n_q_rows,
              "skr_attn_bwd: row range [%d,%d) outside [0,%d)", g->row_begin, g->row_end, n_q_rows);
  if (g->n_tiles == 0 && g->row_end == g->row_begin) return SKR_OK;
  SKR_REQUIRE(q && k && v && o && dout && lse && dq && dk && dv && ws, "skr_attn_bwd: null pointer");
  SKR_REQUIRE(g->cu_seqlens_q && g->q_pos && g->k_start && g->k_len && (g->tiles || g->n_tiles == 0),
              "skr_attn_bwd: null segment table");
  const size_t need = skr_attn_bwd_ws_bytes(s, n_q_rows);
  if (ws_bytes < need) return fail(SKR_E_CAPACITY, "skr_attn_bwd: workspace %zu < %zu bytes", ws_bytes, need);
  if (skr_status e = check_sm100()) return e;
  SKR_REQUIRE(kv_accumulate != 0 || n_kv_rows <= n_q_rows,
              "skr_attn_bwd: kv_accumulate = 0 needs n_kv_rows (%d) <= n_q_rows (%d)", n_kv_rows, n_q_rows);
  AttnArgs a = make_args(s, g, n_q_rows);
  a.peer_dk = peer_dk;
  a.peer_dv = peer_dv;
  a.row_map = row_map;
  a.pad_P = pad_P;
  cudaStream_t st = (cudaStream_t)stream;
  float* Dbuf = (float*)ws;
  float* dk_acc = (float*)((uint8_t*)ws + ws_kv_off(s, n_q_rows));
  float* dv_acc = (float*)((uint8_t*)dk_acc + ws_kv_bytes(s, n_q_rows));
  const int bn = skr_attn_block_n(s), bf16 = s->dtype == SKR_BF16;
  // kv_accumulate = 0: the key tiles split into query bands sum their partials in dk_acc / dv_acc
  if (kv_accumulate == 0)
    if (skr_status e = band_kv(a, bn, s->d, 0, dk_acc, dv_acc, dk, dv, bf16, st)) return e;
  skr_status e;
  if (!bf16) {
    e = simt_attn_bwd(a, s->d, g->row_begin, g->row_end, (const float*)q, (const float*)k, (const float*)v,
                      (const float*)o, (const float*)dout, lse, (float*)dq, (float*)dk, (float*)dv, kv_accumulate,
                      dq_accumulate, Dbuf, dk_acc, dv_acc, st);
  } else {
    float* dq_acc = (float*)((uint8_t*)ws + ws_dq_off(s, n_q_rows));
    e = sm100_attn_bwd(a, s->d, g->row_begin, g->row_end, q, k, v, o, dout, lse, dq, dk, dv, kv_accumulate,
                       dq_accumulate, Dbuf, dq_acc, dk_acc, dv_acc, n_q_rows, n_kv_rows, st);
  }
  if (e) return e;
  if (kv_accumulate == 0) return band_kv(a, bn, s->d, 1, dk_acc, dv_acc, dk, dv, bf16, st);
  return SKR_OK;
}
