// common.cuh -- shared device helpers of libntt (product path only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

// Device-side bounds / invariant checks of the hand-written kernels (compute-sanitizer is not
// available on the GPU pool): a -DNTT_CHECKED build traps with a message on the first violation
// (tests run against it: profiles/checked_r2.md).  Compiled out otherwise.
#ifdef NTT_CHECKED
#include <cstdio>
#define NTT_DCHECK(c)                                                                                  \
  do {                                                                                                 \
    if (!(c)) {                                                                                        \
      printf("NTT_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, blockIdx.x, \
             threadIdx.x);                                                                             \
      __trap();                                                                                        \
    }                                                                                                  \
  } while (0)
#else
#define NTT_DCHECK(c) \
  do {                \
  } while (0)
#endif

namespace ntt {

constexpr int kMaxRank = 64;

// ---------------------------------------------------------------------------
// Counter-based RNG, implemented from the text spec in include/ntt.h
// (ntt_fill_uniform).  u = top 24 bits of mix64(key + (i+1) G) times 2^-24.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t rng_mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__host__ __device__ __forceinline__ uint64_t rng_key(uint64_t seed, uint64_t stream) {
  return rng_mix64(seed ^ rng_mix64(stream + kGolden));
}
__host__ __device__ __forceinline__ float rng_uniform(uint64_t key, uint64_t i) {
  uint32_t v = (uint32_t)(rng_mix64(key + (i + 1ULL) * kGolden) >> 40);
  return (float)v * (1.0f / 16777216.0f);  // exact: v < 2^24
}

__host__ __device__ __forceinline__ uint64_t stream_w(int l) { return 0x200ULL + 2ULL * (uint64_t)l; }
__host__ __device__ __forceinline__ uint64_t stream_h(int l) { return 0x201ULL + 2ULL * (uint64_t)l; }

// MU quotient, reading R4: (w * num) / (den + eps), IEEE division.
__device__ __forceinline__ float mu_quot(float w, float num, float den, float eps) {
  return __fdiv_rn(__fmul_rn(w, num), __fadd_rn(den, eps));
}
__device__ __forceinline__ double mu_quot(double w, double num, double den, double eps) {
  return __ddiv_rn(__dmul_rn(w, num), __dadd_rn(den, eps));
}

// The fp64 MU quotient of the in-kernel W updates, rounded to fp32 by the caller: (w num) /
// (den + eps) through a hardware reciprocal estimate, two Newton steps and one residual
// correction (no call into the IEEE division routine, whose serial slow-path checks dominated the
// persistent kernels' W update).  Within one fp64 ulp of the IEEE quotient, so the fp32 result is
// the IEEE one except when the fp64 quotient lies within an ulp of an fp32 rounding boundary
// (reading R4).  Zero, subnormal, huge or non-finite divisors take the IEEE division.
__device__ __forceinline__ double mu_quot_fast(double w, double num, double den, double eps) {
  const double a = __dmul_rn(w, num), b = __dadd_rn(den, eps);
  if (!(b > 1e-290 && b < 1e290)) return __ddiv_rn(a, b);
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(b));
  double e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  e = fma(-b, r, 1.0);
  r = fma(r, e, r);
  const double q = a * r;
  return fma(r, fma(-b, q, a), q);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// packed fp32x2 FMA (FFMA2 on sm_100a): d = a * b + c lane-wise
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  return __ffma2_rn(a, b, c);
}


// Dynamic shared-memory opt-in of a kernel: raised to the device's per-block maximum, never
// lowered.  Setting it to each call's own size would lower it for later, smaller shapes -- and a
// kernel node captured earlier into a CUDA graph with a larger size then fails when a profiler
// (ncu, per-node graph profiling) re-launches that node against the function's current
// attribute.  The launch's own dynamic size still decides occupancy.
inline cudaError_t smem_optin(const void* kern, size_t bytes) {
  static const int mx = [] {
    int d = 0, v = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    return v;
  }();
  cudaFuncAttributes fa;
  cudaError_t e = cudaFuncGetAttributes(&fa, kern);
  if (e != cudaSuccess) return e;
  const int dyn = mx - (int)fa.sharedSizeBytes;  // the opt-in maximum covers static + dynamic
  if (bytes > (size_t)(dyn > 0 ? dyn : 0)) return cudaErrorInvalidValue;
  if (fa.maxDynamicSharedSizeBytes >= dyn) return cudaSuccess;
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
}

}  // namespace ntt
