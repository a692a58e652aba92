// Throughput probe: legacy warp-level mma.sync m16n8k16 (f16 x f16 -> f32) on B200, and
// ldmatrix.  Not part of the product; decides whether the short-wide fused MU kernels can
// move their contractions onto mma.sync with fp16 hi/lo operand splits.
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>

__global__ void k_mma(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x * 7 + i);
  for (int i = 0; i < 2; ++i) b[i] = 0x3c003c00u ^ (threadIdx.x * 3 + i);
  float c[8][4];
  for (int j = 0; j < 8; ++j)
    for (int i = 0; i < 4; ++i) c[j][i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j)
    for (int i = 0; i < 4; ++i) s += c[j][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ldsm(float* out, int iters) {
  __shared__ __align__(16) unsigned short sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = (unsigned short)i;
  __syncthreads();
  unsigned acc = 0;
  const unsigned base = (unsigned)__cvta_generic_to_shared(sm) + ((threadIdx.x & 31) * 16) + (threadIdx.x >> 5) * 512;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      unsigned r0, r1, r2, r3;
      asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                   : "r"(base + (j & 3) * 2048));
      acc += r0 ^ r1 ^ r2 ^ r3;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)acc;
}

int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * sizeof(float));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int warps : {4, 8, 16}) {
    const int iters = 20000;
    k_mma<<<148, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    k_mma<<<148, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double mmas = 148.0 * warps * iters * 8;
    double macs = mmas * 16 * 8 * 16;
    printf("mma.sync m16n8k16 f16->f32, %2d warps/SM: %.1f MMA/clk/SM (at %d MHz nominal), %.1f TMAC/s\n", warps,
           mmas / 148 / (ms * 1e-3 * clk * 1e3), clk / 1000, macs / (ms * 1e-3) / 1e12);
  }
  for (int warps : {4, 8, 16}) {
    const int iters = 20000;
    k_ldsm<<<148, warps * 32>>>(out, 10);
    cudaEventRecord(e0);
    k_ldsm<<<148, warps * 32>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double n = 148.0 * warps * iters * 8;
    printf("ldmatrix.x4.trans, %2d warps/SM: %.2f instr/clk/SM\n", warps, n / 148 / (ms * 1e-3 * clk * 1e3));
  }
  return 0;
}
