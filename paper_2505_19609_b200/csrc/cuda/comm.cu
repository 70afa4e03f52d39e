// Rows a6 / a9: CP-group collectives over NVLink 5 / NVSwitch (NCCL inside the CP group only).
// Failure detection: skr_comm_wait polls the communicator's asynchronous error state
// while it waits for a stream, and aborts the communicator (which releases NCCL kernels stuck on a
// dead peer) on an error or after a timeout, so a failed rank surfaces as SKR_E_NCCL instead of a
// hung process.
#include <nccl.h>

#include <chrono>
#include <thread>

#include "device.cuh"

struct skr_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
  bool aborted = false;
  cudaEvent_t ev = nullptr;   // skr_comm_wait's marker (created on first use, on the caller's device)
};

namespace {
skr_status nccl_status(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return SKR_OK;
  return skr::fail(SKR_E_NCCL, "%s: %s", what, ncclGetErrorString(r));
}
}  // namespace

SKR_EXPORT int32_t skr_nccl_id_bytes(void) { return (int32_t)sizeof(ncclUniqueId); }

SKR_EXPORT skr_status skr_nccl_get_id(void* id_out) {
  SKR_REQUIRE(id_out, "skr_nccl_get_id: null output");
  ncclUniqueId id;
  if (skr_status s = nccl_status(ncclGetUniqueId(&id), "ncclGetUniqueId")) return s;
  memcpy(id_out, &id, sizeof(id));
  return SKR_OK;
}

SKR_EXPORT skr_status skr_comm_create(const void* nccl_id, int32_t nranks, int32_t rank, skr_comm** out) {
  SKR_REQUIRE(nccl_id && out && nranks >= 1 && rank >= 0 && rank < nranks, "skr_comm_create: bad arguments");
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof(id));
  auto* c = new skr_comm();
  c->nranks = nranks;
  c->rank = rank;
  if (skr_status s = nccl_status(ncclCommInitRank(&c->comm, nranks, id, rank), "ncclCommInitRank")) {
    delete c;
    return s;
  }
  *out = c;
  return SKR_OK;
}

SKR_EXPORT void skr_comm_destroy(skr_comm* c) {
  if (!c) return;
  if (c->comm && !c->aborted) ncclCommDestroy(c->comm);
  if (c->ev) cudaEventDestroy(c->ev);
  delete c;
}

SKR_EXPORT skr_status skr_comm_size(const skr_comm* c, int32_t* nranks, int32_t* rank) {
  SKR_REQUIRE(c && nranks && rank, "skr_comm_size: null argument");
  *nranks = c->nranks;
  *rank = c->rank;
  return SKR_OK;
}

SKR_EXPORT skr_status skr_comm_async_error(skr_comm* c) {
  SKR_REQUIRE(c && c->comm, "skr_comm_async_error: no communicator");
  if (c->aborted) return skr::fail(SKR_E_NCCL, "communicator was aborted");
  ncclResult_t r = ncclSuccess;
  if (skr_status s = nccl_status(ncclCommGetAsyncError(c->comm, &r), "ncclCommGetAsyncError")) return s;
  if (r != ncclSuccess && r != ncclInProgress) return skr::fail(SKR_E_NCCL, "asynchronous NCCL error: %s", ncclGetErrorString(r));
  return SKR_OK;
}

SKR_EXPORT skr_status skr_comm_wait(skr_comm* c, void* stream, double timeout_s) {
  SKR_REQUIRE(c && c->comm && timeout_s > 0, "skr_comm_wait: bad arguments");
  if (c->aborted) return skr::fail(SKR_E_NCCL, "communicator was aborted");
  if (!c->ev && cudaEventCreateWithFlags(&c->ev, cudaEventDisableTiming) != cudaSuccess)
    return skr::fail(SKR_E_CUDA, "skr_comm_wait: event create");
  if (cudaEventRecord(c->ev, (cudaStream_t)stream) != cudaSuccess) return skr::fail(SKR_E_CUDA, "skr_comm_wait: record");
  const auto t0 = std::chrono::steady_clock::now();
  for (int spin = 0;; ++spin) {
    const cudaError_t q = cudaEventQuery(c->ev);
    if (q == cudaSuccess) return SKR_OK;
    if (q != cudaErrorNotReady) return skr::fail(SKR_E_CUDA, "skr_comm_wait: %s", cudaGetErrorString(q));
    ncclResult_t r = ncclSuccess;
    ncclCommGetAsyncError(c->comm, &r);
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if ((r != ncclSuccess && r != ncclInProgress) || el > timeout_s) {
      ncclCommAbort(c->comm);   // unblocks NCCL kernels waiting on a dead peer
      c->aborted = true;
      if (r != ncclSuccess && r != ncclInProgress)
        return skr::fail(SKR_E_NCCL, "rank %d: asynchronous NCCL error: %s (communicator aborted)", c->rank,
                    ncclGetErrorString(r));
      return skr::fail(SKR_E_NCCL, "rank %d: step not done after %.1f s (a peer is dead or stalled; communicator aborted)",
                  c->rank, timeout_s);
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

SKR_EXPORT skr_status skr_comm_all_gather(skr_comm* c, const void* send, void* recv, size_t bytes_per_rank,
                                          void* stream) {
  SKR_REQUIRE(c && c->comm, "skr_comm_all_gather: no communicator");
  if (bytes_per_rank == 0) return SKR_OK;
  SKR_REQUIRE(send && recv, "skr_comm_all_gather: null buffer");
  return nccl_status(ncclAllGather(send, recv, bytes_per_rank, ncclUint8, c->comm, (cudaStream_t)stream),
                     "ncclAllGather");
}

SKR_EXPORT skr_status skr_comm_reduce_scatter_f32(skr_comm* c, const float* send, float* recv, size_t count_per_rank,
                                                  void* stream) {
  SKR_REQUIRE(c && c->comm, "skr_comm_reduce_scatter_f32: no communicator");
  if (count_per_rank == 0) return SKR_OK;
  SKR_REQUIRE(send && recv, "skr_comm_reduce_scatter_f32: null buffer");
  return nccl_status(
      ncclReduceScatter(send, recv, count_per_rank, ncclFloat, ncclSum, c->comm, (cudaStream_t)stream),
      "ncclReduceScatter");
}

SKR_EXPORT skr_status skr_comm_all_reduce_f32(skr_comm* c, float* buf, size_t count, void* stream) {
  SKR_REQUIRE(c && c->comm, "skr_comm_all_reduce_f32: no communicator");
  if (count == 0) return SKR_OK;
  SKR_REQUIRE(buf, "skr_comm_all_reduce_f32: null buffer");
  return nccl_status(ncclAllReduce(buf, buf, count, ncclFloat, ncclSum, c->comm, (cudaStream_t)stream),
                     "ncclAllReduce");
}

// Ring CP (row f4's alternative exchange): one ring hop -- every buffer i is sent to rank + 1
// and recv_bufs[i] receives rank - 1's buffer i, all in one NCCL group (point-to-point over NVLink,
// no collective). A 1-rank communicator sends to itself.
SKR_EXPORT skr_status skr_comm_ring_shift(skr_comm* c, const void* const* send_bufs, void* const* recv_bufs,
                                          const size_t* bytes, int32_t n_bufs, void* stream) {
  SKR_REQUIRE(c && c->comm && n_bufs >= 0 && (n_bufs == 0 || (send_bufs && recv_bufs && bytes)),
              "skr_comm_ring_shift: bad arguments");
  const int next = (c->rank + 1) % c->nranks, prev = (c->rank - 1 + c->nranks) % c->nranks;
  const cudaStream_t st = (cudaStream_t)stream;
  if (skr_status s = nccl_status(ncclGroupStart(), "ncclGroupStart")) return s;
  for (int32_t i = 0; i < n_bufs; ++i) {
    if (bytes[i] == 0) continue;
    if (skr_status s = nccl_status(ncclSend(send_bufs[i], bytes[i], ncclUint8, next, c->comm, st), "ncclSend")) {
      ncclGroupEnd();
      return s;
    }
    if (skr_status s = nccl_status(ncclRecv(recv_bufs[i], bytes[i], ncclUint8, prev, c->comm, st), "ncclRecv")) {
      ncclGroupEnd();
      return s;
    }
  }
  return nccl_status(ncclGroupEnd(), "ncclGroupEnd");
}
