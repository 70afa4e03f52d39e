// fp32 test mode (reading R31): the same varlen causal attention, forward and backward, with
// fp32 inputs/outputs and fp32 FFMA math (one warp per query row or key row). This is the path
// the 1e-5 parity bar of BASELINE.json is checked on; the bf16 path is attn_fwd_sm100.cu /
// attn_bwd_sm100.cu (tcgen05).
#include <cfloat>

#include "attn_common.cuh"
#include "device.cuh"

namespace skr {
namespace simt {

constexpr int kWarps = 8;
constexpr int kRowsPerWarp = 4;
constexpr int kBM = kWarps * kRowsPerWarp;  // 32 query rows per CTA
constexpr int kBN = 32;                     // key tile
constexpr int kMaxD = 128;

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

template <int D>
__global__ void __launch_bounds__(256) fwd_kernel(AttnArgs a, const float* __restrict__ q, const float* __restrict__ k,
                                                  const float* __restrict__ v, float* __restrict__ o,
                                                  float* __restrict__ lse) {
  constexpr int E = D / 32;
  __shared__ float sk[kBN][D], sv[kBN][D];
  const int seg = a.tiles[2 * blockIdx.x], tile = a.tiles[2 * blockIdx.x + 1];
  const int h = blockIdx.y, g = h * a.hkv / a.hq;
  const int cu0 = a.cu[seg], cu1 = a.cu[seg + 1];
  const int qpos = a.q_pos[seg], kst = a.k_start[seg];
  const int r_first = cu0 + tile * kBM;
  const int n_rows = min(kBM, cu1 - r_first);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  float qr[kRowsPerWarp][E], acc[kRowsPerWarp][E], m[kRowsPerWarp], l[kRowsPerWarp];
  int pos[kRowsPerWarp];
#pragma unroll
  for (int i = 0; i < kRowsPerWarp; ++i) {
    const int rr = warp * kRowsPerWarp + i;
    pos[i] = rr < n_rows ? qpos + (r_first + rr - cu0) : -1;
    m[i] = -FLT_MAX;
    l[i] = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      qr[i][e] = rr < n_rows ? q[((size_t)(r_first + rr) * a.hq + h) * D + lane + 32 * e] : 0.f;
      acc[i][e] = 0.f;
    }
  }
  // keys visible to the last row; keys past k_len are invisible (ring CP)
  const int n_keys = min(qpos + (r_first - cu0) + n_rows, a.k_len[seg]);
  for (int kb = 0; kb < n_keys; kb += kBN) {
    __syncthreads();
    for (int idx = threadIdx.x; idx < kBN * D; idx += blockDim.x) {
      const int j = idx / D, c = idx % D;
      const bool ok = kb + j < n_keys;
      const size_t off = ((size_t)(kst + kb + j) * a.hkv + g) * D + c;
      sk[j][c] = ok ? k[off] : 0.f;
      sv[j][c] = ok ? v[off] : 0.f;
    }
    __syncthreads();
    const int jn = min(kBN, n_keys - kb);
    for (int j = 0; j < jn; ++j) {
      const int key = kb + j;
#pragma unroll
      for (int i = 0; i < kRowsPerWarp; ++i) {
        if (key > pos[i]) continue;  // causal (also skips rows past the segment: pos = -1)
        float dot = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) dot += qr[i][e] * sk[j][lane + 32 * e];
        const float s = warp_sum(dot) * a.scale;
        if (s > m[i]) {
          const float alpha = expf(m[i] - s);
          l[i] = l[i] * alpha + 1.f;
#pragma unroll
          for (int e = 0; e < E; ++e) acc[i][e] = acc[i][e] * alpha + sv[j][lane + 32 * e];
          m[i] = s;
        } else {
          const float p = expf(s - m[i]);
          l[i] += p;
#pragma unroll
          for (int e = 0; e < E; ++e) acc[i][e] += p * sv[j][lane + 32 * e];
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < kRowsPerWarp; ++i) {
    const int rr = warp * kRowsPerWarp + i;
    if (rr >= n_rows) continue;
    const size_t row = r_first + rr;
    // a row that sees no key (ring CP): O = 0, LSE = -inf (the merge's neutral element)
    const float inv = l[i] > 0.f ? 1.f / l[i] : 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) o[(row * a.hq + h) * D + lane + 32 * e] = acc[i][e] * inv;
    if (lane == 0) lse[(size_t)h * a.ld_lse + row] = l[i] > 0.f ? m[i] + logf(l[i]) : -INFINITY;
  }
}

// D_i = dO_i . O_i per (row, head); rows [row_begin, row_end).
template <int D>
__global__ void bwd_pre_kernel(int row_begin, int row_end, int hq, const float* __restrict__ o,
                               const float* __restrict__ dout, float* __restrict__ Dbuf, int ld) {
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int row = row_begin + gw / hq, h = gw % hq;
  if (row >= row_end) return;
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < D / 32; ++e) {
    const size_t off = ((size_t)row * hq + h) * D + lane + 32 * e;
    s += o[off] * dout[off];
  }
  s = warp_sum(s);
  if (lane == 0) Dbuf[(size_t)h * ld + row] = s;
}

// dQ: one warp per (query row, head) over rows [row_begin, row_end); segment by binary search.
template <int D>
__global__ void __launch_bounds__(256) bwd_dq_kernel(AttnArgs a, int row_begin, int row_end,
                                                     const float* __restrict__ q, const float* __restrict__ k,
                                                     const float* __restrict__ v, const float* __restrict__ dout,
                                                     const float* __restrict__ lse, const float* __restrict__ Dbuf,
                                                     float* __restrict__ dq, int dq_accumulate) {
  constexpr int E = D / 32;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) / 32, lane = threadIdx.x % 32;
  const int row = row_begin + gw / a.hq, h = gw % a.hq;
  if (row >= row_end) return;
  int lo = 0, hi = a.n_seg;  // find seg with cu[seg] <= row < cu[seg+1]
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (a.cu[mid] <= row) lo = mid; else hi = mid;
  }
  const int seg = lo, g = h * a.hkv / a.hq;
  const int pos = a.q_pos[seg] + row - a.cu[seg];
  float qr[E], dor[E], acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const size_t off = ((size_t)row * a.hq + h) * D + lane + 32 * e;
    qr[e] = q[off];
    dor[e] = dout[off];
    acc[e] = 0.f;
  }
  const float L = lse[(size_t)h * a.ld_lse + row], Di = Dbuf[(size_t)h * a.ld_lse + row];
  const int j_end = min(pos + 1, a.k_len[seg]);
  for (int j = 0; j < j_end; ++j) {
    const size_t ko = ((size_t)(a.k_start[seg] + j) * a.hkv + g) * D;
    float s = 0.f, dp = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      s += qr[e] * k[ko + lane + 32 * e];
      dp += dor[e] * v[ko + lane + 32 * e];
    }
    s = warp_sum(s) * a.scale;
    dp = warp_sum(dp);
    const float p = expf(s - L);
    const float ds = p * (dp - Di);
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] += ds * k[ko + lane + 32 * e];
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    float* d = dq + ((size_t)row * a.hq + h) * D + lane + 32 * e;
    *d = dq_accumulate ? *d + acc[e] * a.scale : acc[e] * a.scale;   // accumulate: ring CP steps
  }
}

// dK, dV: one warp per (key row, kv head), loop over the group's heads and the queries that see it.
template <int D>
__global__ void __launch_bounds__(256) bwd_dkv_kernel(AttnArgs a, const float* __restrict__ q,
                                                      const float* __restrict__ k, const float* __restrict__ v,
                                                      const float* __restrict__ dout, const float* __restrict__ lse,
                                                      const float* __restrict__ Dbuf, float* __restrict__ dk,
                                                      float* __restrict__ dv, int accumulate,
                                                      float* __restrict__ dk_acc, float* __restrict__ dv_acc) {
  constexpr int E = D / 32;
  // work item {seg, key tile, q_lo, q_hi} (skr_tiles_bwd): queries [q_lo, q_hi) of the segment
  const int32_t* item = a.tiles + 4 * blockIdx.x;
  const int seg = item[0], tile = item[1], q_lo = item[2], q_hi = item[3];
  const int g = blockIdx.y, grp = a.hq / a.hkv;
  const int cu0 = a.cu[seg], cu1 = a.cu[seg + 1];
  const int qpos = a.q_pos[seg], qlen = cu1 - cu0, klen = a.k_len[seg];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int per_warp = kBN / kWarps;
  // a band of a split key tile: its partial is added into the band accumulator (locals) or the
  // caller's fp32 accumulator (kv_accumulate 1 / 2)
  const bool partial = q_lo > max(0, tile * kBN - qpos) || q_hi < qlen;
  const int q_end = min(qlen, q_hi);
  for (int i = 0; i < per_warp; ++i) {
    const int j = tile * kBN + warp * per_warp + i;  // key position
    if (j >= klen) break;
    const size_t ko = ((size_t)(a.k_start[seg] + j) * a.hkv + g) * D;
    float kr[E], vr[E], ak[E], av[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      kr[e] = k[ko + lane + 32 * e];
      vr[e] = v[ko + lane + 32 * e];
      ak[e] = av[e] = 0.f;
    }
    const int i0 = max(max(0, j - qpos), q_lo);  // first query (segment-relative) of the item that sees key j
    for (int hh = 0; hh < grp; ++hh) {
      const int h = g * grp + hh;
      for (int r = i0; r < q_end; ++r) {
        const size_t qo = ((size_t)(cu0 + r) * a.hq + h) * D;
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          s += q[qo + lane + 32 * e] * kr[e];
          dp += dout[qo + lane + 32 * e] * vr[e];
        }
        s = warp_sum(s) * a.scale;
        dp = warp_sum(dp);
        const float p = expf(s - lse[(size_t)h * a.ld_lse + cu0 + r]);
        const float ds = p * (dp - Dbuf[(size_t)h * a.ld_lse + cu0 + r]);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          av[e] += p * dout[qo + lane + 32 * e];
          ak[e] += ds * q[qo + lane + 32 * e];
        }
      }
    }
    float* pdk = accumulate == 2 ? peer_row(a, true, a.k_start[seg] + j, g, D) : nullptr;
    float* pdv = accumulate == 2 ? peer_row(a, false, a.k_start[seg] + j, g, D) : nullptr;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (accumulate == 2) {
        atomicAdd(&pdk[lane + 32 * e], ak[e] * a.scale);
        atomicAdd(&pdv[lane + 32 * e], av[e]);
      } else if (accumulate) {
        atomicAdd(&dk[ko + lane + 32 * e], ak[e] * a.scale);
        atomicAdd(&dv[ko + lane + 32 * e], av[e]);
      } else if (partial) {
        atomicAdd(&dk_acc[ko + lane + 32 * e], ak[e] * a.scale);
        atomicAdd(&dv_acc[ko + lane + 32 * e], av[e]);
      } else {
        dk[ko + lane + 32 * e] = ak[e] * a.scale;
        dv[ko + lane + 32 * e] = av[e];
      }
    }
  }
}

}  // namespace simt

skr_status simt_attn_fwd(const AttnArgs& a, int d, const float* q, const float* k, const float* v, float* o,
                         float* lse, cudaStream_t st) {
  if (a.n_tiles == 0) return SKR_OK;
  dim3 grid(a.n_tiles, a.hq);
  if (d == 64)
    simt::fwd_kernel<64><<<grid, 256, 0, st>>>(a, q, k, v, o, lse);
  else if (d == 128)
    simt::fwd_kernel<128><<<grid, 256, 0, st>>>(a, q, k, v, o, lse);
  else if (d == 32)
    simt::fwd_kernel<32><<<grid, 256, 0, st>>>(a, q, k, v, o, lse);
  else
    return fail(SKR_E_UNSUPPORTED, "fp32 mode supports d in {32, 64, 128}");
  return launch_status("simt fwd");
}

skr_status simt_attn_bwd(const AttnArgs& a, int d, int row_begin, int row_end, const float* q, const float* k,
                         const float* v, const float* o, const float* dout, const float* lse, float* dq, float* dk,
                         float* dv, int accumulate, int dq_accumulate, float* Dbuf, float* dk_acc, float* dv_acc,
                         cudaStream_t st) {
  if (row_end > row_begin) {
    const int warps = (row_end - row_begin) * a.hq;
    const int blocks = (warps * 32 + 255) / 256;
    if (d == 64) {
      simt::bwd_pre_kernel<64><<<blocks, 256, 0, st>>>(row_begin, row_end, a.hq, o, dout, Dbuf, a.ld_lse);
      simt::bwd_dq_kernel<64><<<blocks, 256, 0, st>>>(a, row_begin, row_end, q, k, v, dout, lse, Dbuf, dq, dq_accumulate);
    } else if (d == 128) {
      simt::bwd_pre_kernel<128><<<blocks, 256, 0, st>>>(row_begin, row_end, a.hq, o, dout, Dbuf, a.ld_lse);
      simt::bwd_dq_kernel<128><<<blocks, 256, 0, st>>>(a, row_begin, row_end, q, k, v, dout, lse, Dbuf, dq, dq_accumulate);
    } else if (d == 32) {
      simt::bwd_pre_kernel<32><<<blocks, 256, 0, st>>>(row_begin, row_end, a.hq, o, dout, Dbuf, a.ld_lse);
      simt::bwd_dq_kernel<32><<<blocks, 256, 0, st>>>(a, row_begin, row_end, q, k, v, dout, lse, Dbuf, dq, dq_accumulate);
    } else {
      return fail(SKR_E_UNSUPPORTED, "fp32 mode supports d in {32, 64, 128}");
    }
  }
  if (a.n_tiles) {
    dim3 grid(a.n_tiles, a.hkv);
    if (d == 64)
      simt::bwd_dkv_kernel<64><<<grid, 256, 0, st>>>(a, q, k, v, dout, lse, Dbuf, dk, dv, accumulate, dk_acc, dv_acc);
    else if (d == 128)
      simt::bwd_dkv_kernel<128><<<grid, 256, 0, st>>>(a, q, k, v, dout, lse, Dbuf, dk, dv, accumulate, dk_acc, dv_acc);
    else
      simt::bwd_dkv_kernel<32><<<grid, 256, 0, st>>>(a, q, k, v, dout, lse, Dbuf, dk, dv, accumulate, dk_acc, dv_acc);
  }
  return launch_status("simt bwd");
}

}  // namespace skr
