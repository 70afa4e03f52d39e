// C-ABI entry points of the attention kernels (rows a7/a8): argument checks and dispatch.
#include "attn_common.cuh"
#include "device.cuh"

namespace skr {
bool fwd_two_sm();   // attn_fwd_sm100.cu: d = 128 forward on CTA pairs (the libskrull_fwd2sm.so build variant)
skr_status sm100_attn_fwd(const AttnArgs& a, int d, const void* q, const void* k, const void* v, void* o, float* lse,
                          int n_q_rows, int n_kv_rows, cudaStream_t st);
skr_status sm100_attn_bwd(const AttnArgs& a, int d, int row_begin, int row_end, const void* q, const void* k,
                          const void* v, const void* o, const void* dout, const float* lse, void* dq, void* dk,
                          void* dv, int accumulate, float* Dbuf, float* dq_acc, int n_q_rows, int n_kv_rows,
                          cudaStream_t st);

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

SKR_EXPORT size_t skr_attn_bwd_ws_bytes(const skr_attn_shape* s, int32_t n_q_rows) {
  if (!s || n_q_rows < 0) return 0;
  const size_t Dbytes = ((size_t)s->hq * n_q_rows * 4 + 255) & ~size_t(255);
  if (s->dtype == SKR_FP32) return Dbytes;
  return Dbytes + (size_t)n_q_rows * s->hq * s->d * 4;   // + fp32 dQ accumulator
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
                                const int32_t* row_map, int32_t pad_P);

SKR_EXPORT skr_status skr_attn_bwd(const skr_attn_shape* s, const skr_segs* g, const void* q, const void* k,
                                   const void* v, const void* o, const void* dout, const float* lse, void* dq,
                                   void* dk, void* dv, int32_t kv_accumulate, int32_t n_q_rows, int32_t n_kv_rows,
                                   void* ws, size_t ws_bytes, void* stream) {
  SKR_REQUIRE(kv_accumulate == 0 || kv_accumulate == 1, "skr_attn_bwd: kv_accumulate must be 0 or 1");
  return attn_bwd_impl(s, g, q, k, v, o, dout, lse, dq, dk, dv, kv_accumulate, n_q_rows, n_kv_rows, ws, ws_bytes,
                       stream, nullptr, nullptr, nullptr, 0);
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
                                const int32_t* row_map, int32_t pad_P) {
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
  AttnArgs a = make_args(s, g, n_q_rows);
  a.peer_dk = peer_dk;
  a.peer_dv = peer_dv;
  a.row_map = row_map;
  a.pad_P = pad_P;
  cudaStream_t st = (cudaStream_t)stream;
  float* Dbuf = (float*)ws;
  if (s->dtype == SKR_FP32) {
    if (kv_accumulate == 0) {
      // locals: dk/dv rows are written by exactly one segment; fp32 mode writes them directly
    }
    return simt_attn_bwd(a, s->d, g->row_begin, g->row_end, (const float*)q, (const float*)k, (const float*)v,
                         (const float*)o, (const float*)dout, lse, (float*)dq, (float*)dk, (float*)dv, kv_accumulate,
                         Dbuf, st);
  }
  float* dq_acc = (float*)((uint8_t*)ws + (((size_t)s->hq * n_q_rows * 4 + 255) & ~size_t(255)));
  return sm100_attn_bwd(a, s->d, g->row_begin, g->row_end, q, k, v, o, dout, lse, dq, dk, dv, kv_accumulate, Dbuf,
                        dq_acc, n_q_rows, n_kv_rows, st);
}
