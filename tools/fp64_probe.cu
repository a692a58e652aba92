// Probes: dependent-chain latency (1 thread) and one-CTA throughput (288 threads) of fp64 FMA,
// fp64 (x*y)/(x+e), fp32 -> fp64 conversion, FFMA and fp32 IEEE division.  Not part of the product.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x * 1e-9, y = b;
  float xf = (float)a + threadIdx.x * 1e-6f, yf = (float)b;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, y, 0.5);
  __syncthreads();
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = (x * y) / (x + 1e-16);
  __syncthreads();
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) { x += (double)xf; xf = xf * 1.0000001f; }
  __syncthreads();
  long long t3 = clock64();
  for (int i = 0; i < n; ++i) xf = fmaf(xf, yf, 0.5f);
  __syncthreads();
  long long t4 = clock64();
  for (int i = 0; i < n; ++i) xf = (xf * yf) / (xf + 1e-16f);
  __syncthreads();
  long long t5 = clock64();
  out[threadIdx.x] = x + xf;
  if (threadIdx.x == 0) {
    cyc[0] = (t1 - t0) / n; cyc[1] = (t2 - t1) / n; cyc[2] = (t3 - t2) / n; cyc[3] = (t4 - t3) / n; cyc[4] = (t5 - t4) / n;
  }
}
int main() {
  double* o; long long* c;
  cudaMalloc(&o, 8 * 1024); cudaMallocManaged(&c, 64);
  for (int th : {1, 32, 288}) {
    k<<<1, th>>>(o, c, 1.0001, 0.9999, 1000);
    cudaDeviceSynchronize();
    k<<<1, th>>>(o, c, 1.0001, 0.9999, 1000);
    cudaDeviceSynchronize();
    printf("%3d threads, cycles per iteration: DFMA %lld  fp64 (x*y)/(x+e) %lld  x += (double)f %lld  FFMA %lld  fp32 div %lld\n",
           th, c[0], c[1], c[2], c[3], c[4]);
  }
  return 0;
}
