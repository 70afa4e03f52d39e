// Building-block self-test: one 128 x n x 128 bf16 UMMA through each operand layout the
// attention kernels use (TMA SW128 K-major, TMA SW128 MN-major, thread-written SW128 K-major).
#include "device.cuh"
#include "sm100.cuh"
#include "tma.h"

namespace skr {

// smem: A 32 KB (two 64-wide chunks of 128 rows), B 32 KB, barriers.
__global__ void __launch_bounds__(128, 1)
    selftest_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                    const __nv_bfloat16* __restrict__ A, float* __restrict__ C, int variant, int n, int reps,
                    long long* cycles, int chains) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + 32768;
  uint64_t* bar_tma = reinterpret_cast<uint64_t*>(smem + 65536);
  uint64_t* bar_mma = bar_tma + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_tma + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (threadIdx.x == 0) {
    mbar_init(bar_tma, 1);
    mbar_init(bar_mma, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc<512>(tmem_slot);
  // variant 3: A [128][128] written by threads into SW128 K-major smem (as P is in attention)
  if (variant == 3) {
    const int row = threadIdx.x;
    for (int c = 0; c < 128; c += 8) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(A + row * 128 + c);
      uint32_t base = smem_u32(sA + (c / 64) * 16384);
      st_shared_v4(base + sw128_off(row, c % 64), src[0], src[1], src[2], src[3]);
    }
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // variant 4: A [128][128] written by threads into TMEM columns [128, 192) as packed bf16 pairs
  if (variant == 4) {
    const int row = threadIdx.x;
    for (int c = 0; c < 64; c += 32) {
      uint32_t r[32];
      const uint32_t* src = reinterpret_cast<const uint32_t*>(A + row * 128 + 2 * c);
      for (int i = 0; i < 32; ++i) r[i] = src[i];
      tmem_st32(tmem + ((uint32_t)(warp * 32) << 16) + 128 + c, r);
    }
    tmem_wait_st();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
  }

  if (warp == 0) {
    // warp-converged issue loop; one elected lane issues (operands stay warp-uniform)
    const bool a_tma = variant != 3 && variant != 4;
    const bool b_mn = variant == 1 || variant == 2;
    const bool a_mn = variant == 2;
    uint32_t bytes = (a_tma ? 32768u : 0u) + (uint32_t)n * 256u;
    if (elect_one()) {
      mbar_expect_tx(bar_tma, bytes);
      for (int ch = 0; ch < 2; ++ch) {
        if (a_tma) tma_load_2d(sA + ch * 16384, &ta, bar_tma, ch * 64, 0);  // 64 cols x 128 rows
      }
      if (b_mn) {
        // B global [K=128][n]: chunks of 64 n-columns x 128 K-rows
        for (int ch = 0; ch < n / 64; ++ch) tma_load_2d(sB + ch * 16384, &tb, bar_tma, ch * 64, 0);
      } else {
        // B global [n][K=128]: chunks of 64 K-columns x n rows
        for (int ch = 0; ch < 2; ++ch) tma_load_2d(sB + ch * (n * 128), &tb, bar_tma, ch * 64, 0);
      }
    }
    __syncwarp();
    mbar_wait(bar_tma, 0);
    tc_fence_after();
    const uint32_t idesc = idesc_bf16_f32(128, n, a_mn ? 1 : 0, b_mn ? 1 : 0);
    const uint32_t sa = smem_u32(sA), sb = smem_u32(sB);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      ad[k] = a_mn ? sdesc_sw128(sa + k * 2048, 16384, 1024) : sdesc_sw128(sa + (k / 4) * 16384 + (k % 4) * 32, 16, 1024);
      bd[k] = b_mn ? sdesc_sw128(sb + k * 2048, 16384, 1024)
                   : sdesc_sw128(sb + (k / 4) * (n * 128) + (k % 4) * 32, 16, 1024);
    }
    const long long t0 = clock64();
    if (chains < 0) {
      // latency mode: groups of -chains MMAs, each followed by commit + wait (serialised groups)
      const int g = -chains;
      uint32_t ph = 1;   // bar_mma phase 0 is used by the final commit below; start at phase 1 parity
      uint64_t* bar2 = bar_mma + 2;
      if (elect_one()) mbar_init(bar2, 1);
      __syncwarp();
      fence_mbar_init();
      ph = 0;
      for (int rep = 0; rep < reps; ++rep) {
        if (elect_one()) {
          for (int k = 0; k < g; ++k) umma_f16(tmem, ad[k & 7], bd[k & 7], idesc, k > 0);
          umma_commit(bar2);
        }
        __syncwarp();
        mbar_wait(bar2, ph);
        ph ^= 1;
        tc_fence_after();
      }
    } else if (chains >= 200) {
      // issue-path probe mode (chains = 200 + m): `reps` warp-converged groups of 4 MMAs, each group
      // committed to bar2 (never waited), then m = 0 nothing, 1 mbarrier probe of an idle barrier,
      // 2 probe of bar2 itself, 3 a plain shared-memory load, 4 probe of an idle barrier without
      // the commit. Cycles of the whole sequence (does a barrier probe wait for the committed MMAs?)
      const int m = (chains - 200) % 10;
      const int gs = (chains - 200) / 10 == 1 ? 8 : (chains - 200) / 10 == 2 ? 2 : 4;   // MMAs per group
      uint64_t* bar2 = bar_mma + 2;
      uint64_t* bar3 = bar_mma + 3;
      if (elect_one()) { mbar_init(bar2, 1); mbar_init(bar3, 1); }
      __syncwarp();
      fence_mbar_init();
      int acc = 0;
      volatile int* vs = reinterpret_cast<volatile int*>(bar_mma + 4);
      if (m == 6) {
        // control: the same groups + commits, all inside one elected region (no per-group election)
        if (elect_one()) {
          for (int rep = 0; rep < reps; ++rep) {
#pragma unroll
            for (int k = 0; k < 4; ++k) umma_f16(tmem, ad[k], bd[k], idesc, k > 0 || rep > 0);
            umma_commit(bar2);
          }
        }
        __syncwarp();
      }
      for (int rep = 0; rep < (m == 6 ? 0 : reps); ++rep) {
        if (elect_one()) {
          if (m == 5) {
            // descriptors formed inside the issue block from the shared-memory bases (uniform values)
            const uint64_t a0 = sdesc_sw128(sa, 16, 1024), b0 = sdesc_sw128(sb, 16, 1024);
#pragma unroll
            for (int k = 0; k < 4; ++k)
              umma_f16(tmem, a0 + (uint64_t)(((k / 4) * 16384 + (k % 4) * 32) >> 4),
                       b0 + (uint64_t)(((k / 4) * (n * 128) + (k % 4) * 32) >> 4), idesc, k > 0 || rep > 0);
          } else if (gs == 2) {
#pragma unroll
            for (int k = 0; k < 2; ++k) umma_f16(tmem, ad[k], bd[k], idesc, k > 0 || rep > 0);
          } else if (gs == 4) {
#pragma unroll
            for (int k = 0; k < 4; ++k) umma_f16(tmem, ad[k], bd[k], idesc, k > 0 || rep > 0);
          } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) umma_f16(tmem, ad[k], bd[k], idesc, k > 0 || rep > 0);
          }
          if (m != 4) umma_commit(bar2);
        }
        __syncwarp();
        if (m == 1 || m == 4) acc += __shfl_sync(0xffffffffu, mbar_test(bar3, 0) ? 1 : 0, 0);
        else if (m == 2) acc += __shfl_sync(0xffffffffu, mbar_test(bar2, rep & 1) ? 1 : 0, 0);
        else if (m == 3) acc += vs[lane];
      }
      if (lane == 0 && cycles) cycles[1] = acc;   // mode 2: how many probes found their own group complete
    } else if (chains >= 100) {
      // mixed-stream mode (chains = 100 + m): m = 0 SS/TS alternating into one accumulator,
      // m = 1 SS N=n / SS N=64 alternating idesc into two accumulators, m = 2 SS into 2 accumulators,
      // m = 3 TS/SS alternating into two accumulators
      const int m = chains - 100;
      const uint32_t id64 = idesc_bf16_f32(128, 64, a_mn ? 1 : 0, b_mn ? 1 : 0);
      if (elect_one()) {
        for (int rep = 0; rep < reps; ++rep)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (m == 0) {
              if (k & 1) umma_f16_ts(tmem, tmem + 128 + k * 8, bd[k], idesc, 1);
              else umma_f16(tmem, ad[k], bd[k], idesc, k > 0);
            } else if (m == 1) {
              if (k & 1) umma_f16(tmem + 256, ad[k], bd[k], id64, k > 1);
              else umma_f16(tmem, ad[k], bd[k], idesc, k > 0);
            } else if (m == 2) {
              umma_f16(tmem + (k & 1) * 256, ad[k], bd[k], idesc, k > 1);
            } else {
              if (k & 1) umma_f16_ts(tmem + 256, tmem + 128 + k * 8, bd[k], idesc, k > 1);
              else umma_f16(tmem, ad[k], bd[k], idesc, k > 0);
            }
          }
      }
      __syncwarp();
    } else
    // one elected lane issues the whole MMA stream (descriptors precomputed, warp-uniform)
    if (elect_one()) {
      if (variant == 4) {
        for (int rep = 0; rep < reps; ++rep)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t dcol = chains > 1 ? (uint32_t)((k % chains) * n) : 0u;
            umma_f16_ts(tmem + dcol, tmem + 128 + k * 8, bd[k], idesc, chains > 1 ? (k >= chains) : (k > 0));
          }
      } else {
        for (int rep = 0; rep < reps; ++rep)
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t dcol = chains > 1 ? (uint32_t)((k % chains) * n) : 0u;
            umma_f16(tmem + dcol, ad[k], bd[k], idesc, chains > 1 ? (k >= chains) : (k > 0));
          }
      }
    }
    __syncwarp();
    if (elect_one()) umma_commit(bar_mma);
    __syncwarp();
    if (cycles) {
      mbar_wait(bar_mma, 0);
      if (lane == 0) cycles[0] = clock64() - t0;
    }
  }
  __syncwarp();
  mbar_wait(bar_mma, 0);
  tc_fence_after();
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < n; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c0, r);
    tmem_wait_ld();
    for (int i = 0; i < 32; ++i) C[row * n + c0 + i] = __uint_as_float(r[i]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

}  // namespace skr

SKR_EXPORT skr_status skr_selftest_umma(int32_t variant, int32_t n, const void* A, const void* B, float* C,
                                         void* stream) {
  using namespace skr;
  if (skr_status s = check_sm100()) return s;
  SKR_REQUIRE(variant >= 0 && variant <= 4 && (n == 64 || n == 128) && A && B && C, "bad selftest args");
  CUtensorMap ta, tb;
  const bool b_mn = variant == 1 || variant == 2;
  // A: K-major [128][128] (variants 0,1) or MN-major given as [K=128][M=128] (variant 2): same shape.
  if (!make_tmap_2d(&ta, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 128, 128, 128, 128, 64, true))
    return fail(SKR_E_CUDA, "tensor map A");
  if (b_mn) {
    if (!make_tmap_2d(&tb, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 128, n, n, 128, 64, true))
      return fail(SKR_E_CUDA, "tensor map B");
  } else {
    if (!make_tmap_2d(&tb, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n, 128, 128, n, 64, true))
      return fail(SKR_E_CUDA, "tensor map B");
  }
  const int smem = 65536 + 64 + 1024;
  cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  selftest_kernel<<<1, 128, smem, (cudaStream_t)stream>>>(ta, tb, (const __nv_bfloat16*)A, C, variant, n, 1,
                                                           nullptr, 1);
  return launch_status("selftest_kernel");
}

// Debug aid: cycles for `reps` x 8 UMMAs (128 x n x 16 each) of operand layout `variant` on one SM.
extern "C" __attribute__((visibility("default"))) int skr_debug_umma_cycles(int variant, int n, int reps,
                                                                           const void* A, const void* B,
                                                                           float* C, long long* cycles,
                                                                           int chains) {
  using namespace skr;
  CUtensorMap ta, tb;
  const bool b_mn = variant == 1 || variant == 2;
  make_tmap_2d(&ta, A, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 128, 128, 128, 128, 64, true);
  if (b_mn)
    make_tmap_2d(&tb, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, 128, n, n, 128, 64, true);
  else
    make_tmap_2d(&tb, B, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, n, 128, 128, n, 64, true);
  const int smem = 65536 + 1024 + 1024;   // + barriers / probe words of the debug modes
  cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  selftest_kernel<<<1, 128, smem>>>(ta, tb, (const __nv_bfloat16*)A, C, variant, n, reps, cycles, chains);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}

// Debug aid: MUFU ex2 throughput. `warps` warps (one CTA, one SM) each run `iters` x 16 independent
// ex2.approx (8 chains); mode 1 interleaves each ex2 with one FFMA2 + FADD2 + F2FP (the softmax mix).
namespace skr {
__global__ void mufu_kernel(int iters, int mode, long long* cycles, float* sink) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = 0.001f * (threadIdx.x + i);
  uint32_t pk = 0;
  float2 acc = make_float2(0.f, 0.f);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      if (mode == 1) {
        const float2 xx = ffma2(make_float2(x[i], x[i + 1]), make_float2(0.5f, 0.5f), make_float2(-0.25f, -0.25f));
        x[i] = ex2(xx.x);
        x[i + 1] = ex2(xx.y);
        acc = fadd2(acc, make_float2(x[i], x[i + 1]));
        pk ^= pack_bf16(x[i], x[i + 1]);
      } else if (mode == 2 || mode == 3) {
        // packed half-precision ex2: two results per instruction (mode 2 f16x2, mode 3 bf16x2)
        uint32_t h = __float_as_uint(x[i]);
        if (mode == 2)
          asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(h));
        else
          asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(h));
        x[i] = __uint_as_float(h ^ 0x80008000u);
        x[i + 1] = x[i];
      } else {
        x[i] = ex2(x[i] * -0.5f);
        x[i + 1] = ex2(x[i + 1] * -0.5f);
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
  float s = acc.x + acc.y + (float)pk;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += x[i];
  if (s == 12345.f) sink[0] = s;
}
}  // namespace skr

extern "C" __attribute__((visibility("default"))) int skr_debug_mufu_cycles(int warps, int iters, int mode,
                                                                           long long* cycles, float* sink) {
  skr::mufu_kernel<<<1, warps * 32>>>(iters, mode, cycles, sink);
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : 1;
}
