// Rows a6 / a9: CP-group collectives over NVLink 5 / NVSwitch (NCCL inside the CP group only).
#include <nccl.h>

#include "device.cuh"

struct skr_comm {
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
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
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
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
