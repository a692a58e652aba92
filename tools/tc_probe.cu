// Throughput / latency probe for tcgen05.mma kind::tf32 with small N on B200.
// Not part of the product.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//   -I paper_2008_01340_b200/csrc tools/tc_probe.cu -o tools/tc_probe -lcuda
#include <cstdio>
#include <cuda_runtime.h>

#include "sm100.cuh"
using namespace ntt::sm100;

// one CTA per SM; one thread issues `iters` x `per` MMAs of shape M=128 x N (SS)
// into `nacc` rotating accumulators, then commits and waits.  Returns cycles.
template <int N, bool TS>
__global__ void k_probe(int iters, int nacc, long long* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.001f * (i & 255);
  if (warp == 0) tmem_alloc(&slot, 512);
  if (threadIdx.x == 32) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = slot;
  if (threadIdx.x == 32) {
    const uint32_t sa = smem_u32(sm), sb = sa + 16384;
    const uint32_t id = idesc_tf32(128, N, false, false);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t d = tb + (uint32_t)((it * 4 + kk) % nacc) * N;
        const uint64_t bd = umma_desc_sw128(sb + kk * 32, 16, 1024);
        if (TS)
          mma_tf32_ts(d, tb + 256 + kk * 8, bd, id, 1u);
        else
          mma_tf32_ss(d, umma_desc_sw128(sa + kk * 32, 16, 1024), bd, id, 1u);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tb, 512);
  }
}

template <int N, bool TS>
void run(const char* name, int nacc) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * 148);
  cudaFuncSetAttribute(k_probe<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384 + 32768);
  const int iters = 4096;
  k_probe<N, TS><<<148, 128, 16384 + 32768>>>(iters, nacc, d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < 148; ++i) cyc += h[i];
  cyc /= 148;
  const double mmas = iters * 4.0;
  printf("%-22s N=%3d nacc=%d: %.1f cycles/MMA, %.0f MAC/clk/SM  (%s)\n", name, N, nacc, cyc / mmas,
         128.0 * N * 8 * mmas / cyc, cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  for (int nacc : {1, 2, 4}) {
    run<8, false>("SS", nacc);
    run<16, false>("SS", nacc);
    run<32, false>("SS", nacc);
    run<64, false>("SS", nacc);
    run<128, false>("SS", nacc);
    run<16, true>("TS", nacc);
    run<32, true>("TS", nacc);
    run<64, true>("TS", nacc);
  }
  return 0;
}
