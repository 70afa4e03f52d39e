// Arguments shared by the attention kernels (fp32 SIMT test mode and bf16 tcgen05).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../common.h"

namespace skr {

struct AttnArgs {
  const int32_t* cu;       // [n_seg+1] packed query rows
  const int32_t* q_pos;    // [n_seg]
  const int32_t* k_start;  // [n_seg]
  const int32_t* k_len;    // [n_seg]
  const int32_t* tiles;    // fwd [2*n_tiles] {seg, tile}; bwd [4*n_tiles] {seg, key tile, q_lo, q_hi}
  int n_seg, n_tiles;
  int hq, hkv;
  float scale;
  int ld_lse;              // row stride of lse / D buffers ([h][ld_lse])
  // backward with kv_accumulate == 2 (row f3, fused peer reduction): dK / dV fp32 partials are
  // red-added straight into each key row's OWNER accumulator: owner = row_map[k] / pad_P, row
  // row_map[k] % pad_P of the [pad_P][hkv][d] fp32 buffers at peer_dk[owner] / peer_dv[owner]
  const uint64_t* peer_dk = nullptr;
  const uint64_t* peer_dv = nullptr;
  const int32_t* row_map = nullptr;   // [natural K rows] -> owner * pad_P + row in the owner's prefix
  int pad_P = 0;
};

// destination of KV head g's dK / dV partial row in accumulate mode 2 (see AttnArgs): the owner's
// accumulator row prow, head g, d fp32 values
__device__ __forceinline__ float* peer_row(const AttnArgs& a, bool is_dk, int krow, int g, int d) {
  const int gr = a.row_map[krow];
  const int owner = gr / a.pad_P, prow = gr - owner * a.pad_P;
  return reinterpret_cast<float*>(is_dk ? a.peer_dk[owner] : a.peer_dv[owner]) + ((size_t)prow * a.hkv + g) * d;
}

skr_status simt_attn_fwd(const AttnArgs& a, int d, const float* q, const float* k, const float* v, float* o,
                         float* lse, cudaStream_t st);
skr_status simt_attn_bwd(const AttnArgs& a, int d, int row_begin, int row_end, const float* q, const float* k,
                         const float* v, const float* o, const float* dout, const float* lse, float* dq, float* dk,
                         float* dv, int accumulate, int dq_accumulate, float* Dbuf, float* dk_acc, float* dv_acc,
                         cudaStream_t st);

}  // namespace skr
