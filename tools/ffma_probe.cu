// Throughput probe: FFMA (3-reg) vs FFMA2 per SM on B200.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ffma(float* out, float a, float b, int iters) {
  float x[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) x[i] = threadIdx.x * 0.001f + i;
  float y = b + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(x[i], y, a + i * 0.f + x[(i + 1) & 15] * 0.f);
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma_reg(float* out, float a, float b, int iters) {
  float x[16], c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { x[i] = threadIdx.x * 0.001f + i; c[i] = a * i + threadIdx.x; }
  float y = b + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = fmaf(c[i], y, x[i]);
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fmaf(x[i], y, c[i]);
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += x[i] + c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b, int iters) {
  float2 x[16], c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) { x[i] = make_float2(threadIdx.x * 0.001f + i, i); c[i] = make_float2(a * i, threadIdx.x); }
  float y = b + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = __ffma2_rn(make_float2(y, y), c[i], x[i]);
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = __ffma2_rn(make_float2(y, y), x[i], c[i]);
  }
  float s = 0; for (int i = 0; i < 16; ++i) s += x[i].x + c[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out; cudaMalloc(&out, sizeof(float) * sms * 8 * 256);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000; dim3 grid(sms * 4), block(256);
  for (int rep = 0; rep < 2; ++rep) {
    float ms;
    cudaEventRecord(e0); k_ffma_reg<<<grid, block>>>(out, 1.0001f, 0.9999f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double f = 2.0 * 32 * iters * (double)grid.x * block.x;
    printf("FFMA  : %.1f TFLOP/s (%.1f FMA/clk/SM @1965)\n", f / ms / 1e9, f / 2 / (ms * 1e-3) / sms / 1.965e9);
    cudaEventRecord(e0); k_ffma2<<<grid, block>>>(out, 1.0001f, 0.9999f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    f = 2.0 * 64 * iters * (double)grid.x * block.x;
    printf("FFMA2 : %.1f TFLOP/s (%.1f FMA/clk/SM @1965)\n", f / ms / 1e9, f / 2 / (ms * 1e-3) / sms / 1.965e9);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
