// shared-memory load throughput by access pattern (wavefront cost of broadcast LDS.128 / LDS.32)
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void __launch_bounds__(512) k(float* out, int iters) {
  __shared__ __align__(16) float s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0.001f;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  float4 acc = make_float4(0, 0, 0, 0);
  int off;
  if (MODE == 0) off = 0;                      // LDS128 uniform
  else if (MODE == 1) off = (lane & 7) * 4;    // LDS128 8 distinct x4 (phase-A pattern)
  else if (MODE == 2) off = lane * 4;          // LDS128 32 distinct
  else if (MODE == 3) off = lane;              // LDS32 32 distinct
  else off = 0;                                // LDS32 uniform
  for (int it = 0; it < iters; ++it) {
    const int base = (it & 31) * 128;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE <= 2) {
        float4 v = *reinterpret_cast<const float4*>(&s[(base + u * 128 + off) & 4095]);
        acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
      } else {
        float v = s[(base + u * 128 + off) & 4095];
        acc.x += v;
      }
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == -1.f) out[0] = acc.x;
}
template <int MODE> void run(const char* name, float* d) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096;
  k<MODE><<<148 * 2, 512>>>(d, iters);
  cudaEventRecord(a);
  k<MODE><<<148 * 2, 512>>>(d, iters);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double warp_loads = 148.0 * 2 * 16 * iters * 8;
  printf("%-28s %.3f ms  %.2f warp-loads/clk/SM (at 1.9GHz)\n", name, ms, warp_loads / (ms * 1e-3 * 1.9e9) / 148);
}
int main() {
  float* d; cudaMalloc(&d, 64);
  run<0>("LDS128 uniform", d); run<1>("LDS128 8 distinct x4", d); run<2>("LDS128 32 distinct", d);
  run<3>("LDS32 32 distinct", d); run<4>("LDS32 uniform", d);
  return 0;
}
