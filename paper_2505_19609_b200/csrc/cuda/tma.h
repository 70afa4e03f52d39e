// Host-side TMA tensor-map construction (driver entry point, no -lcuda).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

namespace skr {

// 2-D bf16 (or fp32) tensor map over a row-major matrix [rows][cols] with row stride
// `row_stride_elems`, box [box_rows][box_cols], 128-byte swizzle (box_cols*elem == 128 B)
// or no swizzle. Out-of-bounds rows read as zero. Returns false on failure.
bool make_tmap_2d(CUtensorMap* map, const void* base, CUtensorMapDataType dtype, int elem_bytes, uint64_t rows,
                  uint64_t cols, uint64_t row_stride_elems, uint32_t box_rows, uint32_t box_cols, bool swizzle128);

}  // namespace skr
