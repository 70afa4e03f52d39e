// Row f3 (first step): the CP exchange as peer-memory kernels instead of NCCL collectives.
//
// Every rank of a CP group maps the other ranks' buffers into its address space (CUDA IPC; over
// NVLink / NVSwitch the loads and stores below travel as peer accesses) and:
//   a6  peer gather : copies each distributed chunk's K/V rows straight from its OWNER's packed
//                     buffer into this rank's natural distributed-K/V buffer -- the all-gather, its
//                     [N][P] staging buffer and the reorder pass become one pass (Eq. 5 volume only).
//   a9  peer reduce : for each chunk this rank owns, sums the fp32 dK/dV partials of all ranks
//                     (read from their natural buffers) and writes bf16 into its packed dK/dV prefix
//                     -- permute + reduce-scatter + cast become one pass.
// Ordering between ranks uses per-rank epoch flags: `signal` stores the epoch into this rank's slot
// of every peer's flag array (release, system scope, after a system fence); `wait` spins with
// acquire loads until every slot reached the epoch (bounded: it gives up after ~10 s and raises an
// error word instead of hanging the GPU).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "device.cuh"

namespace skr {

int chunk_blocks_x(int n_chunks);   // movement.cu

// chunk table rows: {seq, chunk, owner, gathered_row, natural_row, len}
__global__ void peer_gather_kernel(const uint64_t* __restrict__ peer_base, const int32_t* __restrict__ table,
                                   int n_chunks, int vpr, int pad_rows_P, uint4* __restrict__ natural) {
  for (int ch = blockIdx.y; ch < n_chunks; ch += gridDim.y) {
    const int32_t* t = table + 6 * ch;
    const int owner = t[2];
    const int64_t src_row = t[3] - (int64_t)owner * pad_rows_P, n = t[4], len = t[5];
    const uint4* __restrict__ src = reinterpret_cast<const uint4*>(peer_base[owner]) + src_row * vpr;
    uint4* __restrict__ dst = natural + n * vpr;
    const int64_t total = len * vpr;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x)
      dst[i] = src[i];
  }
}

template <bool kBf16>
__global__ void peer_reduce_kernel(const uint64_t* __restrict__ peer_base, int nranks, int rank,
                                   const int32_t* __restrict__ table, int n_chunks, int v4pr, int pad_rows_P,
                                   void* __restrict__ dst) {
  for (int ch = blockIdx.y; ch < n_chunks; ch += gridDim.y) {
    const int32_t* t = table + 6 * ch;
    if (t[2] != rank) continue;                        // only the chunks this rank owns
    const int64_t drow = t[3] - (int64_t)rank * pad_rows_P, n = t[4], len = t[5];
    const int64_t total = len * v4pr;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
      float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int r = 0; r < nranks; ++r) {               // fixed rank order: deterministic sums
        const float4 v = reinterpret_cast<const float4*>(peer_base[r])[n * v4pr + i];
        acc.x += v.x, acc.y += v.y, acc.z += v.z, acc.w += v.w;
      }
      if (kBf16) {
        __nv_bfloat162 a = __floats2bfloat162_rn(acc.x, acc.y), b = __floats2bfloat162_rn(acc.z, acc.w);
        uint2 o;
        o.x = *reinterpret_cast<uint32_t*>(&a);
        o.y = *reinterpret_cast<uint32_t*>(&b);
        reinterpret_cast<uint2*>(dst)[drow * v4pr + i] = o;
      } else {
        reinterpret_cast<float4*>(dst)[drow * v4pr + i] = acc;
      }
    }
  }
}

__global__ void peer_signal_kernel(const uint64_t* __restrict__ peer_flags, int nranks, int rank, uint32_t epoch) {
  __threadfence_system();                             // this stream's earlier writes before the flag
  for (int n = threadIdx.x; n < nranks; n += blockDim.x) {
    uint32_t* f = reinterpret_cast<uint32_t*>(peer_flags[n]) + rank;
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f), "r"(epoch) : "memory");
  }
}

__global__ void peer_wait_kernel(const uint32_t* __restrict__ flags, int nranks, uint32_t epoch, int32_t* err) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int n = threadIdx.x; n < nranks; n += blockDim.x) {
    while (true) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + n) : "memory");
      if ((int32_t)(v - epoch) >= 0) break;
      uint64_t t1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
      if (t1 - t0 > 10000000000ull) {                  // 10 s: a peer never signalled
        atomicExch(err, 1);
        break;
      }
      __nanosleep(200);
    }
  }
}

// ---- IPC export / import of device buffers (interior pointers of a caching allocator's segment)
using PFN_getRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
static PFN_getRange get_range_fn() {
  static PFN_getRange fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_getRange>(p);
  });
  return fn;
}

struct Mapped {
  void* base;
  int refs;
};
static std::mutex g_ipc_mu;
static std::map<std::string, Mapped> g_ipc;   // handle bytes -> mapping (one open per handle per process)

}  // namespace skr

using namespace skr;

static const int kBlob = (int)(sizeof(cudaIpcMemHandle_t) + sizeof(int64_t));

SKR_EXPORT int32_t skr_ipc_blob_bytes(void) { return kBlob; }

SKR_EXPORT skr_status skr_ipc_export(const void* ptr, void* blob_out) {
  SKR_REQUIRE(ptr && blob_out, "skr_ipc_export: null pointer");
  auto fn = get_range_fn();
  if (!fn) return fail(SKR_E_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (fn(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return fail(SKR_E_CUDA, "cuMemGetAddressRange failed");
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, (void*)base) != cudaSuccess) return fail(SKR_E_CUDA, "cudaIpcGetMemHandle failed");
  const int64_t off = (int64_t)((CUdeviceptr)ptr - base);
  memcpy(blob_out, &h, sizeof(h));
  memcpy((uint8_t*)blob_out + sizeof(h), &off, sizeof(off));
  return SKR_OK;
}

SKR_EXPORT skr_status skr_ipc_import(const void* blob, void** ptr_out) {
  SKR_REQUIRE(blob && ptr_out, "skr_ipc_import: null pointer");
  cudaIpcMemHandle_t h;
  int64_t off;
  memcpy(&h, blob, sizeof(h));
  memcpy(&off, (const uint8_t*)blob + sizeof(h), sizeof(off));
  const std::string key((const char*)&h, sizeof(h));
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  auto it = g_ipc.find(key);
  if (it == g_ipc.end()) {
    void* base = nullptr;
    if (cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
      return fail(SKR_E_CUDA, "cudaIpcOpenMemHandle failed");
    it = g_ipc.emplace(key, Mapped{base, 0}).first;
  }
  it->second.refs++;
  *ptr_out = (uint8_t*)it->second.base + off;
  return SKR_OK;
}

SKR_EXPORT skr_status skr_ipc_close_all(void) {
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  for (auto& kv : g_ipc) cudaIpcCloseMemHandle(kv.second.base);
  g_ipc.clear();
  return SKR_OK;
}

SKR_EXPORT skr_status skr_peer_gather_chunks(const uint64_t* peer_packed, const int32_t* chunk_table,
                                             int32_t n_chunks, int32_t row_bytes, int32_t pad_rows_P, void* natural,
                                             void* stream) {
  SKR_REQUIRE(n_chunks >= 0 && row_bytes > 0 && row_bytes % 16 == 0 && pad_rows_P >= 0,
              "skr_peer_gather_chunks: bad sizes");
  if (n_chunks == 0) return SKR_OK;
  SKR_REQUIRE(peer_packed && chunk_table && natural, "skr_peer_gather_chunks: null pointer");
  if (skr_status e = check_sm100()) return e;
  dim3 grid(chunk_blocks_x(n_chunks), std::min(n_chunks, 65535));
  peer_gather_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(peer_packed, chunk_table, n_chunks, row_bytes / 16,
                                                            pad_rows_P, (uint4*)natural);
  return launch_status("peer_gather_chunks");
}

SKR_EXPORT skr_status skr_peer_reduce_chunks(const uint64_t* peer_partials, int32_t nranks, int32_t rank,
                                             const int32_t* chunk_table, int32_t n_chunks, int32_t row_elems,
                                             int32_t pad_rows_P, void* dst, int32_t dst_bf16, void* stream) {
  SKR_REQUIRE(nranks >= 1 && rank >= 0 && rank < nranks && n_chunks >= 0 && row_elems > 0 && row_elems % 4 == 0 &&
                  pad_rows_P >= 0,
              "skr_peer_reduce_chunks: bad sizes");
  if (n_chunks == 0) return SKR_OK;
  SKR_REQUIRE(peer_partials && chunk_table && dst, "skr_peer_reduce_chunks: null pointer");
  if (skr_status e = check_sm100()) return e;
  // only the chunks this rank owns (about 1/nranks of them) do work: size the blocks per chunk for those
  dim3 grid(chunk_blocks_x(std::max(1, n_chunks / nranks)), std::min(n_chunks, 65535));
  if (dst_bf16)
    peer_reduce_kernel<true><<<grid, 256, 0, (cudaStream_t)stream>>>(peer_partials, nranks, rank, chunk_table,
                                                                     n_chunks, row_elems / 4, pad_rows_P, dst);
  else
    peer_reduce_kernel<false><<<grid, 256, 0, (cudaStream_t)stream>>>(peer_partials, nranks, rank, chunk_table,
                                                                      n_chunks, row_elems / 4, pad_rows_P, dst);
  return launch_status("peer_reduce_chunks");
}

SKR_EXPORT skr_status skr_peer_signal(const uint64_t* peer_flags, int32_t nranks, int32_t rank, uint32_t epoch,
                                      void* stream) {
  SKR_REQUIRE(peer_flags && nranks >= 1 && rank >= 0 && rank < nranks, "skr_peer_signal: bad arguments");
  if (skr_status e = check_sm100()) return e;
  peer_signal_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(peer_flags, nranks, rank, epoch);
  return launch_status("peer_signal");
}

SKR_EXPORT skr_status skr_peer_wait(const uint32_t* flags, int32_t nranks, uint32_t epoch, int32_t* err,
                                    void* stream) {
  SKR_REQUIRE(flags && err && nranks >= 1, "skr_peer_wait: bad arguments");
  if (skr_status e = check_sm100()) return e;
  peer_wait_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(flags, nranks, epoch, err);
  return launch_status("peer_wait");
}
