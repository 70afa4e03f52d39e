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
  const int32_t* tiles;    // [2*n_tiles] {seg, tile}
  int n_seg, n_tiles;
  int hq, hkv;
  float scale;
  int ld_lse;              // row stride of lse / D buffers ([h][ld_lse])
};

skr_status simt_attn_fwd(const AttnArgs& a, int d, const float* q, const float* k, const float* v, float* o,
                         float* lse, cudaStream_t st);
skr_status simt_attn_bwd(const AttnArgs& a, int d, int row_begin, int row_end, const float* q, const float* k,
                         const float* v, const float* o, const float* dout, const float* lse, float* dq, float* dk,
                         float* dv, int accumulate, float* Dbuf, cudaStream_t st);

}  // namespace skr
