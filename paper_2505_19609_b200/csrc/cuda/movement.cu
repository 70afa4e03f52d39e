// Rows a5 / a6 / a9: HBM-bound data movement of the CP step.
//   pack      dst[r] = src[src_row[r]]                    (rank-natural -> packed order)
//   unpack    dst[src_row[r]] = src[r]                    (packed -> rank-natural order)
//   gather    rank-major all-gather output -> natural distributed order, per chunk table
//   scatter   natural fp32 partials -> rank-major [N][P] reduce-scatter input (padding zeroed)
//   cast      fp32 -> bf16
// Rows are moved as 16-byte vectors; a warp streams consecutive vectors of one row, so every
// request is a fully used 128-byte line. Grids are multiples of the SM count (grid-stride loops).
#include <cuda_bf16.h>

#include "device.cuh"

namespace skr {

// Blocks per chunk for the chunk-table kernels (grid.y = chunks): enough that the whole grid is
// ~8 blocks per SM however few chunks there are (one 128K sequence over CP=2 has 4 chunks).
int chunk_blocks_x(int n_chunks) {
  const int y = std::max(1, std::min(n_chunks, 65535));
  return std::max(1, std::min(4096, (sm_count() * 8 + y - 1) / y));
}

static int grid_for(int64_t work_items, int threads) {
  int64_t need = (work_items + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * 8;
  return (int)std::max<int64_t>(1, std::min(need, cap));
}

// (row, column) of flat vector index i in rows of vpr vectors: 32-bit division whenever the whole
// index space fits (always at this path's sizes: a 128K-row chunk of 1 KB rows is 8M vectors);
// a 64-bit div / mod per 16-byte vector is a slow software sequence on the GPU
template <typename Index>
__device__ __forceinline__ void row_col(Index i, int vpr, int64_t& r, int64_t& c) {
  const Index q = i / (Index)vpr;
  r = (int64_t)q;
  c = (int64_t)(i - q * (Index)vpr);
}

template <typename Index>
__global__ void pack_rows_kernel(const uint4* __restrict__ src, const int32_t* __restrict__ src_row, int64_t n_rows,
                                 int vpr, uint4* __restrict__ dst, int inverse) {
  const Index total = (Index)(n_rows * vpr);
  for (Index i = blockIdx.x * (Index)blockDim.x + threadIdx.x; i < total; i += (Index)gridDim.x * blockDim.x) {
    int64_t r, c;
    row_col<Index>(i, vpr, r, c);
    const int64_t s = src_row[r];
    if (inverse)
      dst[s * vpr + c] = src[r * vpr + c];
    else
      dst[r * vpr + c] = src[s * vpr + c];
  }
}

// chunk table rows: {seq, chunk, owner, gathered_row, natural_row, len} (skr_pack_chunks layout:
// per distributed sequence in plan order, its 2N chunks c = 0 .. 2N-1)
// to_natural = 1: gathered [N][P] -> natural (a6 reorder). to_natural = 0: natural -> rank-major
// [N][P] (a9 permute); there grid.y also covers `cp` extra items that zero each rank slot's padding
// rows [end_r, P) -- the reduce-scatter sums them, so they must be finite -- and nothing else
// (owner r's prefix ends with chunk 2N-1-r of the last distributed sequence, R21).
__global__ void chunks_kernel(const uint4* __restrict__ from, const int32_t* __restrict__ table, int n_chunks, int vpr,
                              uint4* __restrict__ to, int to_natural, int cp, int pad_rows_P) {
  const int n_items = n_chunks + (to_natural ? 0 : cp);
  for (int ch = blockIdx.y; ch < n_items; ch += gridDim.y) {
    int64_t g, n, len;
    if (ch < n_chunks) {
      const int32_t* t = table + 6 * ch;
      g = t[3], n = t[4], len = t[5];
    } else {                                           // padding rows of rank slot r
      const int r = ch - n_chunks;
      const int32_t* t = table + 6 * (n_chunks - 2 * cp + (2 * cp - 1 - r));
      const int64_t end = (int64_t)t[3] + t[5];        // one past owner r's last row
      g = end, n = 0, len = (int64_t)(r + 1) * pad_rows_P - end;
    }
    const bool small = len * vpr < (int64_t)INT32_MAX;
    const int64_t total = len * vpr;
    if (small) {
      for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < (uint32_t)total; i += gridDim.x * blockDim.x) {
        int64_t r, c;
        row_col<uint32_t>(i, vpr, r, c);
        if (ch >= n_chunks)
          to[(g + r) * vpr + c] = make_uint4(0u, 0u, 0u, 0u);
        else if (to_natural)
          to[(n + r) * vpr + c] = from[(g + r) * vpr + c];
        else
          to[(g + r) * vpr + c] = from[(n + r) * vpr + c];
      }
    } else {
      for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r, c;
        row_col<int64_t>(i, vpr, r, c);
        if (ch >= n_chunks)
          to[(g + r) * vpr + c] = make_uint4(0u, 0u, 0u, 0u);
        else if (to_natural)
          to[(n + r) * vpr + c] = from[(g + r) * vpr + c];
        else
          to[(g + r) * vpr + c] = from[(n + r) * vpr + c];
      }
    }
  }
}

__global__ void cast_kernel(const float4* __restrict__ src, uint2* __restrict__ dst, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&a);
    o.y = *reinterpret_cast<uint32_t*>(&b);
    dst[i] = o;
  }
}

}  // namespace skr

using namespace skr;

SKR_EXPORT skr_status skr_pack_rows(const void* src, const int32_t* src_row, int32_t n_rows, int32_t row_bytes,
                                    void* dst, void* stream) {
  SKR_REQUIRE(n_rows >= 0 && row_bytes > 0 && row_bytes % 16 == 0, "skr_pack_rows: row_bytes must be a multiple of 16");
  if (n_rows == 0) return SKR_OK;
  SKR_REQUIRE(src && src_row && dst, "skr_pack_rows: null pointer");
  if (skr_status e = check_sm100()) return e;
  const int vpr = row_bytes / 16;
  if ((int64_t)n_rows * vpr < (int64_t)INT32_MAX)
    pack_rows_kernel<uint32_t><<<grid_for((int64_t)n_rows * vpr, 256), 256, 0, (cudaStream_t)stream>>>(
        (const uint4*)src, src_row, n_rows, vpr, (uint4*)dst, 0);
  else
    pack_rows_kernel<int64_t><<<grid_for((int64_t)n_rows * vpr, 256), 256, 0, (cudaStream_t)stream>>>(
        (const uint4*)src, src_row, n_rows, vpr, (uint4*)dst, 0);
  return launch_status("pack_rows");
}

SKR_EXPORT skr_status skr_unpack_rows(const void* src, const int32_t* src_row, int32_t n_rows, int32_t row_bytes,
                                      void* dst, void* stream) {
  SKR_REQUIRE(n_rows >= 0 && row_bytes > 0 && row_bytes % 16 == 0, "skr_unpack_rows: row_bytes must be a multiple of 16");
  if (n_rows == 0) return SKR_OK;
  SKR_REQUIRE(src && src_row && dst, "skr_unpack_rows: null pointer");
  if (skr_status e = check_sm100()) return e;
  const int vpr = row_bytes / 16;
  if ((int64_t)n_rows * vpr < (int64_t)INT32_MAX)
    pack_rows_kernel<uint32_t><<<grid_for((int64_t)n_rows * vpr, 256), 256, 0, (cudaStream_t)stream>>>(
        (const uint4*)src, src_row, n_rows, vpr, (uint4*)dst, 1);
  else
    pack_rows_kernel<int64_t><<<grid_for((int64_t)n_rows * vpr, 256), 256, 0, (cudaStream_t)stream>>>(
        (const uint4*)src, src_row, n_rows, vpr, (uint4*)dst, 1);
  return launch_status("unpack_rows");
}

SKR_EXPORT skr_status skr_gather_chunks(const void* gathered, const int32_t* chunk_table, int32_t n_chunks,
                                        int32_t row_bytes, void* natural, void* stream) {
  SKR_REQUIRE(n_chunks >= 0 && row_bytes > 0 && row_bytes % 16 == 0, "skr_gather_chunks: bad sizes");
  if (n_chunks == 0) return SKR_OK;
  SKR_REQUIRE(gathered && chunk_table && natural, "skr_gather_chunks: null pointer");
  if (skr_status e = check_sm100()) return e;
  dim3 grid(chunk_blocks_x(n_chunks), std::min(n_chunks, 65535));
  chunks_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>((const uint4*)gathered, chunk_table, n_chunks, row_bytes / 16,
                                                        (uint4*)natural, 1, 0, 0);
  return launch_status("gather_chunks");
}

SKR_EXPORT skr_status skr_scatter_chunks(const void* natural, const int32_t* chunk_table, int32_t n_chunks,
                                         int32_t row_bytes, int32_t pad_rows_P, int32_t cp, void* rankmajor,
                                         void* stream) {
  SKR_REQUIRE(n_chunks >= 0 && row_bytes > 0 && row_bytes % 16 == 0 && pad_rows_P >= 0 && cp >= 1,
              "skr_scatter_chunks: bad sizes");
  if (pad_rows_P == 0) return SKR_OK;
  SKR_REQUIRE(natural && rankmajor && (chunk_table || n_chunks == 0), "skr_scatter_chunks: null pointer");
  if (skr_status e = check_sm100()) return e;
  cudaStream_t st = (cudaStream_t)stream;
  // rows of a rank's slot beyond its own distributed rows are never read by the owner, but the
  // reduce-scatter sums them: the same launch zeroes exactly those padding rows (cp extra items)
  if (n_chunks == 0) return cuda_status(cudaMemsetAsync(rankmajor, 0, (size_t)cp * pad_rows_P * row_bytes, st),
                                        "scatter memset");
  SKR_REQUIRE(n_chunks % (2 * cp) == 0, "skr_scatter_chunks: chunk table is not skr_pack_chunks' (2N rows per sequence)");
  const int items = n_chunks + cp;
  dim3 grid(chunk_blocks_x(items), std::min(items, 65535));
  chunks_kernel<<<grid, 256, 0, st>>>((const uint4*)natural, chunk_table, n_chunks, row_bytes / 16,
                                      (uint4*)rankmajor, 0, cp, pad_rows_P);
  return launch_status("scatter_chunks");
}

SKR_EXPORT skr_status skr_cast_f32_bf16(const float* src, void* dst, int64_t n, void* stream) {
  SKR_REQUIRE(n >= 0 && n % 4 == 0, "skr_cast_f32_bf16: n must be a multiple of 4");
  if (n == 0) return SKR_OK;
  SKR_REQUIRE(src && dst, "skr_cast_f32_bf16: null pointer");
  if (skr_status e = check_sm100()) return e;
  cast_kernel<<<grid_for(n / 4, 256), 256, 0, (cudaStream_t)stream>>>((const float4*)src, (uint2*)dst, n / 4);
  return launch_status("cast_f32_bf16");
}
