// Row a8: packed varlen causal attention backward on sm_100a (tcgen05). [in progress]
#include "attn_common.cuh"
#include "device.cuh"

namespace skr {

skr_status sm100_attn_bwd(const AttnArgs& a, int d, int row_begin, int row_end, const void* q, const void* k,
                          const void* v, const void* o, const void* dout, const float* lse, void* dq, void* dk,
                          void* dv, int accumulate, float* Dbuf, float* dq_acc, int n_q_rows, int n_kv_rows,
                          cudaStream_t st) {
  return fail(SKR_E_UNSUPPORTED, "bf16 backward not built yet");
}

}  // namespace skr
