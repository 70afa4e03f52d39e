// a1: Skrull's performance model (Appendix C).
#include <cmath>
#include <cstdint>

#include "../common.h"

namespace skr {

// Eq. 12 in 128-bit: 20 b h^2 S + 4 b h h_kv S + 4 b h S^2.
bool flops128(int64_t S, const skr_model& m, __int128* out) {
  if (S < 0 || m.hidden < 0 || m.kv_hidden < 0 || m.pack_batch < 0) return false;
  const __int128 b = m.pack_batch, h = m.hidden, hkv = m.kv_hidden, s = S;
  *out = 20 * b * h * h * s + 4 * b * h * hkv * s + 4 * b * h * s * s;
  return true;
}

}  // namespace skr

using skr::fail;

SKR_EXPORT skr_status skr_flops(int64_t S, const skr_model* m, int64_t* out) {
  SKR_REQUIRE(m && out && S >= 0, "skr_flops: null argument or negative length");
  __int128 f;
  if (!skr::flops128(S, *m, &f)) return fail(SKR_E_ARG, "skr_flops: negative model field");
  if (f > (__int128)INT64_MAX) return fail(SKR_E_OVERFLOW, "skr_flops: FLOPs(%lld) exceeds int64", (long long)S);
  *out = (int64_t)f;
  return SKR_OK;
}

SKR_EXPORT skr_status skr_volume(int64_t S, const skr_model* m, int64_t* out) {
  SKR_REQUIRE(m && out && S >= 0, "skr_volume: null argument or negative length");
  const __int128 v = (__int128)m->pack_batch * S * m->kv_hidden;   // Eq. 14
  if (v > (__int128)INT64_MAX) return fail(SKR_E_OVERFLOW, "skr_volume overflow");
  *out = (int64_t)v;
  return SKR_OK;
}

SKR_EXPORT double skr_t_comp(double flops, const skr_fit* fit) {   // Eq. 13, R36
  if (!fit || flops == 0.0) return 0.0;
  return fit->slope * flops + fit->intercept;
}

SKR_EXPORT double skr_t_comm(double volume, const skr_fit* fit) {  // Eq. 15, R26
  if (!fit || volume == 0.0) return 0.0;
  return fit->slope * volume + fit->intercept;
}

SKR_EXPORT skr_status skr_fit_linear(const double* x, const double* y, int32_t n, double min_x, skr_fit* out) {
  SKR_REQUIRE(out && (n == 0 || (x && y)) && n >= 0, "skr_fit_linear: bad arguments");
  // Ordinary least squares over the points at/above the threshold.
  double sx = 0, sy = 0;
  int k = 0;
  for (int i = 0; i < n; ++i)
    if (x[i] >= min_x) sx += x[i], sy += y[i], ++k;
  if (k < 2) return fail(SKR_E_PROFILE, "skr_fit_linear: %d qualifying points (< 2)", k);
  const double mx = sx / k, my = sy / k;
  double sxx = 0, sxy = 0;
  for (int i = 0; i < n; ++i)
    if (x[i] >= min_x) sxx += (x[i] - mx) * (x[i] - mx), sxy += (x[i] - mx) * (y[i] - my);
  if (sxx == 0) return fail(SKR_E_PROFILE, "skr_fit_linear: all x equal");
  out->slope = sxy / sxx;
  out->intercept = my - out->slope * mx;
  if (out->intercept < 0) out->intercept = 0;
  return SKR_OK;
}

SKR_EXPORT skr_status skr_bucket_size(double budget, const skr_fit* mem, int64_t* C) {
  SKR_REQUIRE(mem && C, "skr_bucket_size: null argument");
  // Appendix C.1: Memory(S) = alpha S + beta  =>  C = floor((budget - beta) / alpha)
  if (!(budget > mem->intercept) || !(mem->slope > 0))
    return fail(SKR_E_BUDGET, "skr_bucket_size: budget %.6g <= beta %.6g (or alpha <= 0)", budget, mem->intercept);
  *C = (int64_t)std::floor((budget - mem->intercept) / mem->slope);
  return SKR_OK;
}
