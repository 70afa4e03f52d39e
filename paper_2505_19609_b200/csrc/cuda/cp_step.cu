// Rows a5-a9 as one C-ABI call per direction: the CP-rank step of one micro-batch (SURVEY.md §8(b)
// skr_cp_attn_fwd / skr_cp_attn_bwd), sequenced natively on a main and a side stream.
//
// Forward (Eq. 2 executed literally):
//   main : pack Q, K, V (a5)                                     -> ev_packed
//   side : wait ev_packed; all-gather the K/V distributed prefix (a6, NCCL inside the CP group);
//          reorder rank-major -> natural distributed order        -> ev_kv
//   main : attention fwd over LOCAL segments (overlaps the exchange); wait ev_kv;
//          attention fwd over DISTRIBUTED chunks (a7)
// Backward (mirror, reading R24):
//   main : pack dO; zero the fp32 partials; attention bwd over DISTRIBUTED chunks (a8) -> ev_dkv
//   side : wait ev_dkv; permute natural -> rank-major, reduce-scatter (sum), cast into the packed
//          dK/dV distributed prefix (a9)                          -> ev_rs
//   main : attention bwd over LOCAL segments (overlaps the exchange); wait ev_rs
// With no distributed sequence no collective is issued (T_comm(0) = 0, R26) and comm may be null.
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: named ranges for nsys / ncu --nvtx (SURVEY §5 tracing)

#include "attn_common.cuh"
#include "device.cuh"

struct skr_attn_plan {
  skr_attn_shape shape;
  int32_t max_rows;
};

namespace {

struct Events {   // per host thread and device: the two cross-stream hand-overs of a call
  cudaEvent_t a = nullptr, b = nullptr;
};
// events belong to the device that was current when they were created: keyed by device ordinal
Events& events() {
  thread_local Events ev[64];
  int dev = 0;
  cudaGetDevice(&dev);
  Events& e = ev[(dev >= 0 && dev < 64) ? dev : 0];
  if (!e.a) {
    cudaEventCreateWithFlags(&e.a, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&e.b, cudaEventDisableTiming);
  }
  return e;
}

skr_status check_step(const skr_attn_plan* plan, const skr_cp_step* st, skr_comm* comm, const char* who) {
  SKR_REQUIRE(plan && st, "%s: null plan / step", who);
  SKR_REQUIRE(st->cp >= 1 && st->rows >= 0 && st->buf_rows >= st->rows && st->buf_rows >= st->pad_rows_P &&
                  st->buf_rows <= plan->max_rows && st->dist_rows >= 0 && st->dist_rows <= st->rows &&
                  st->natural_rows >= 0 && st->n_chunks >= 0,
              "%s: inconsistent sizes (rows %d, buffer %d, plan max %d, P %d)", who, st->rows, st->buf_rows,
              plan->max_rows, st->pad_rows_P);
  SKR_REQUIRE(st->natural_rows == 0 || comm, "%s: distributed chunks need a communicator", who);
  if (comm && st->natural_rows > 0) {
    int32_t n = 0, r = 0;
    if (skr_status e = skr_comm_size(comm, &n, &r)) return e;
    SKR_REQUIRE(n == st->cp, "%s: step planned for CP = %d but the communicator has %d ranks", who, st->cp, n);
  }
  return SKR_OK;
}

// optional per-call timing (skr_cp_step.timing_events)
skr_status mark(const skr_cp_step* st, int i, cudaStream_t m) {
  if (!st->timing_events) return SKR_OK;
  return skr::cuda_status(cudaEventRecord((cudaEvent_t)st->timing_events[i], m), "record timing event");
}

// NVTX range scoped to a C-ABI phase (host-side markers around the enqueue of each row's work;
// free when no tool is attached)
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
};

size_t row_bytes(const skr_attn_shape& s, int heads) {
  return (size_t)heads * s.d * (s.dtype == SKR_FP32 ? 4 : 2);
}

}  // namespace

using namespace skr;

SKR_EXPORT skr_status skr_attn_plan_create(const skr_attn_shape* s, int32_t max_rows, skr_attn_plan** out) {
  SKR_REQUIRE(s && out && max_rows >= 0, "skr_attn_plan_create: bad arguments");
  SKR_REQUIRE(s->hq >= 1 && s->hkv >= 1 && s->hq % s->hkv == 0, "skr_attn_plan_create: hq must be a multiple of hkv");
  *out = new skr_attn_plan{*s, max_rows};
  return SKR_OK;
}

SKR_EXPORT void skr_attn_plan_destroy(skr_attn_plan* p) { delete p; }

SKR_EXPORT skr_status skr_cp_attn_fwd(skr_comm* comm, const skr_attn_plan* plan, const skr_cp_step* st, void* main,
                                      void* side) {
  if (skr_status e = check_step(plan, st, comm, "skr_cp_attn_fwd")) return e;
  Range r_all("skr_cp_attn_fwd");
  const skr_attn_shape& s = plan->shape;
  const bool dist = st->natural_rows > 0;
  cudaStream_t m = (cudaStream_t)main, sd = (cudaStream_t)side;
  Events& ev = events();
  if (st->rows) {   // a5
    Range r("a5 pack Q/K/V");
    if (skr_status e = skr_pack_rows(st->q_src, st->src_row, st->rows, (int32_t)row_bytes(s, s.hq), st->q, m)) return e;
    if (skr_status e = skr_pack_rows(st->k_src, st->src_row, st->rows, (int32_t)row_bytes(s, s.hkv), st->k, m)) return e;
    if (skr_status e = skr_pack_rows(st->v_src, st->src_row, st->rows, (int32_t)row_bytes(s, s.hkv), st->v, m)) return e;
  }
  if (dist) {       // a6 on the side stream
    Range r("a6 all-gather + reorder (side stream)");
    const size_t kvb = row_bytes(s, s.hkv);
    if (skr_status e = cuda_status(cudaEventRecord(ev.a, m), "record packed")) return e;
    if (skr_status e = cuda_status(cudaStreamWaitEvent(sd, ev.a, 0), "wait packed")) return e;
    if (ncclGroupStart() != ncclSuccess) return fail(SKR_E_NCCL, "ncclGroupStart");
    skr_status e1 = skr_comm_all_gather(comm, st->k, st->k_gathered, (size_t)st->pad_rows_P * kvb, sd);
    skr_status e2 = skr_comm_all_gather(comm, st->v, st->v_gathered, (size_t)st->pad_rows_P * kvb, sd);
    if (ncclGroupEnd() != ncclSuccess) return fail(SKR_E_NCCL, "ncclGroupEnd");
    if (e1) return e1;
    if (e2) return e2;
    if (skr_status e = skr_gather_chunks(st->k_gathered, st->chunk_table, st->n_chunks, (int32_t)kvb, st->k_natural, sd))
      return e;
    if (skr_status e = skr_gather_chunks(st->v_gathered, st->chunk_table, st->n_chunks, (int32_t)kvb, st->v_natural, sd))
      return e;
    if (skr_status e = cuda_status(cudaEventRecord(ev.b, sd), "record kv")) return e;
  }
  // a7: locals first (they need no exchange), then the distributed chunks
  Range r7("a7 attention fwd");
  if (skr_status e = mark(st, 0, m)) return e;
  if (skr_status e = skr_attn_fwd(&s, &st->local_fwd, st->q, st->k, st->v, st->o, st->lse, st->buf_rows, st->buf_rows, m))
    return e;
  if (skr_status e = mark(st, 1, m)) return e;
  if (dist) {
    if (skr_status e = cuda_status(cudaStreamWaitEvent(m, ev.b, 0), "wait kv")) return e;
  }
  if (skr_status e = mark(st, 2, m)) return e;
  if (dist) {
    if (skr_status e = skr_attn_fwd(&s, &st->dist_fwd, st->q, st->k_natural, st->v_natural, st->o, st->lse,
                                    st->buf_rows, st->natural_rows, m))
      return e;
  }
  return mark(st, 3, m);
}

SKR_EXPORT skr_status skr_cp_attn_bwd(skr_comm* comm, const skr_attn_plan* plan, const skr_cp_step* st, void* main,
                                      void* side) {
  if (skr_status e = check_step(plan, st, comm, "skr_cp_attn_bwd")) return e;
  Range r_all("skr_cp_attn_bwd");
  const skr_attn_shape& s = plan->shape;
  const bool dist = st->natural_rows > 0;
  cudaStream_t m = (cudaStream_t)main, sd = (cudaStream_t)side;
  Events& ev = events();
  if (st->rows) {
    if (skr_status e = skr_pack_rows(st->do_src, st->src_row, st->rows, (int32_t)row_bytes(s, s.hq), st->dout, m))
      return e;
  }
  if (dist) {       // a8 distributed chunks first, then a9 on the side stream
    const size_t kv_elems = (size_t)st->natural_rows * s.hkv * s.d;
    if (skr_status e = cuda_status(cudaMemsetAsync(st->dk_partial, 0, kv_elems * 4, m), "zero dK partial")) return e;
    if (skr_status e = cuda_status(cudaMemsetAsync(st->dv_partial, 0, kv_elems * 4, m), "zero dV partial")) return e;
  }
  if (skr_status e = mark(st, 4, m)) return e;
  if (dist) {
    Range r("a8 attention bwd, distributed chunks");
    if (skr_status e = skr_attn_bwd(&s, &st->dist_bwd, st->q, st->k_natural, st->v_natural, st->o, st->dout, st->lse,
                                    st->dq, st->dk_partial, st->dv_partial, 1, st->buf_rows, st->natural_rows, st->ws,
                                    st->ws_bytes, m))
      return e;
  }
  if (skr_status e = mark(st, 5, m)) return e;
  if (dist) {
    Range r("a9 permute + reduce-scatter + cast (side stream)");
    if (skr_status e = cuda_status(cudaEventRecord(ev.a, m), "record partials")) return e;
    if (skr_status e = cuda_status(cudaStreamWaitEvent(sd, ev.a, 0), "wait partials")) return e;
    const int32_t f32b = (int32_t)((size_t)s.hkv * s.d * 4);
    if (skr_status e = skr_scatter_chunks(st->dk_partial, st->chunk_table, st->n_chunks, f32b, st->pad_rows_P, st->cp,
                                          st->dk_rankmajor, sd))
      return e;
    if (skr_status e = skr_scatter_chunks(st->dv_partial, st->chunk_table, st->n_chunks, f32b, st->pad_rows_P, st->cp,
                                          st->dv_rankmajor, sd))
      return e;
    const size_t per_rank = (size_t)st->pad_rows_P * s.hkv * s.d;
    if (ncclGroupStart() != ncclSuccess) return fail(SKR_E_NCCL, "ncclGroupStart");
    skr_status e1 = skr_comm_reduce_scatter_f32(comm, st->dk_rankmajor, st->dk_reduced, per_rank, sd);
    skr_status e2 = skr_comm_reduce_scatter_f32(comm, st->dv_rankmajor, st->dv_reduced, per_rank, sd);
    if (ncclGroupEnd() != ncclSuccess) return fail(SKR_E_NCCL, "ncclGroupEnd");
    if (e1) return e1;
    if (e2) return e2;
    if (st->dist_rows) {
      const size_t n = (size_t)st->dist_rows * s.hkv * s.d;
      if (s.dtype == SKR_FP32) {
        if (skr_status e = cuda_status(cudaMemcpyAsync(st->dk, st->dk_reduced, n * 4, cudaMemcpyDeviceToDevice, sd),
                                       "dK copy"))
          return e;
        if (skr_status e = cuda_status(cudaMemcpyAsync(st->dv, st->dv_reduced, n * 4, cudaMemcpyDeviceToDevice, sd),
                                       "dV copy"))
          return e;
      } else {
        if (skr_status e = skr_cast_f32_bf16(st->dk_reduced, st->dk, (int64_t)n, sd)) return e;
        if (skr_status e = skr_cast_f32_bf16(st->dv_reduced, st->dv, (int64_t)n, sd)) return e;
      }
    }
    if (skr_status e = cuda_status(cudaEventRecord(ev.b, sd), "record rs")) return e;
  }
  Range r8("a8 attention bwd, local segments");
  if (skr_status e = mark(st, 6, m)) return e;
  if (skr_status e = skr_attn_bwd(&s, &st->local_bwd, st->q, st->k, st->v, st->o, st->dout, st->lse, st->dq, st->dk,
                                  st->dv, 0, st->buf_rows, st->buf_rows, st->ws, st->ws_bytes, m))
    return e;
  if (skr_status e = mark(st, 7, m)) return e;
  if (dist) {
    if (skr_status e = cuda_status(cudaStreamWaitEvent(m, ev.b, 0), "wait rs")) return e;
  }
  return SKR_OK;
}
