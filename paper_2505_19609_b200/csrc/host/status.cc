// Status strings and the thread-local last-error message (skrull.h conventions).
#include "../common.h"

#include <cstring>

namespace skr {

static thread_local char g_err[512] = {0};

skr_status fail(skr_status s, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return s;
}

void clear_error() { g_err[0] = 0; }

}  // namespace skr

SKR_EXPORT const char* skr_status_string(skr_status s) {
  switch (s) {
    case SKR_OK: return "ok";
    case SKR_E_ARG: return "invalid argument";
    case SKR_E_SCHEDULE: return "DACP scheduling failed (roll-back impossible or disabled)";
    case SKR_E_GDS: return "GDS found no feasible micro-batching";
    case SKR_E_BUDGET: return "memory budget below the fitted intercept";
    case SKR_E_PROFILE: return "insufficient profile points";
    case SKR_E_OVERFLOW: return "integer overflow";
    case SKR_E_CAPACITY: return "caller buffer too small";
    case SKR_E_CUDA: return "CUDA error";
    case SKR_E_NCCL: return "NCCL error";
    case SKR_E_UNSUPPORTED: return "unsupported device or shape";
    default: return "unknown status";
  }
}

SKR_EXPORT const char* skr_last_error(void) { return skr::g_err; }

SKR_EXPORT int32_t skr_abi_version(void) { return 2; }   // 2: cp_step, attn_plan, peer exchange
