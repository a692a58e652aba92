// tmabench.cu -- read bandwidth of 1-D bulk copies (cp.async.bulk) into a shared-memory ring
// (tools only): one producer lane per CTA streams `rows` row segments of `seg` bytes per stage,
// NC consumer warps wait for the stage and release it (no compute).  Prints GB/s.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tmabench tools/tmabench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_tma(const float* __restrict__ X, long long n, int rows, int seg_floats, int ns, int nc) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ns; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(nc));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const long long ntiles = n / seg_floats;
  const uint32_t stage_bytes = (uint32_t)rows * seg_floats * 4;
  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        // wait empty (parity ph ^ 1)
        asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(
                         su32(&empty[s])), "r"(ph ^ 1u)
                     : "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage_bytes) : "memory");
        for (int i = 0; i < rows; ++i) {
          const float* src = X + (long long)i * n + t * seg_floats;
          unsigned char* dst = sm + (size_t)s * stage_bytes + (size_t)i * seg_floats * 4;
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(dst)),
                       "l"(src), "r"((uint32_t)seg_floats * 4), "r"(su32(&full[s]))
                       : "memory");
        }
        if (++s == ns) { s = 0; ph ^= 1u; }
      }
    }
  } else if (warp <= nc) {
    int s = 0;
    uint32_t ph = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) {
      asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" ::"r"(su32(&full[s])),
                   "r"(ph)
                   : "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
      if (++s == ns) { s = 0; ph ^= 1u; }
    }
  }
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 10077696;
  const int rows = argc > 2 ? atoi(argv[2]) : 11;
  const int seg = argc > 3 ? atoi(argv[3]) : 448;
  const int ns = argc > 4 ? atoi(argv[4]) : 8;
  const int nc = 4;
  float* X;
  cudaMalloc(&X, sizeof(float) * n * rows);
  cudaMemset(X, 1, sizeof(float) * n * rows);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = (size_t)ns * rows * seg * 4;
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 2; ++w) k_tma<<<sms, (nc + 1) * 32, smem>>>(X, n, rows, seg, ns, nc);
  cudaEventRecord(a);
  const int reps = 10;
  for (int it = 0; it < reps; ++it) k_tma<<<sms, (nc + 1) * 32, smem>>>(X, n, rows, seg, ns, nc);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  const double bytes = 4.0 * (double)(n / seg * seg) * rows;
  printf("rows=%d seg=%d B (%d floats) stages=%d stage=%zu B : %.1f GB/s %s\n", rows, seg * 4, seg, ns, smem / ns,
         bytes / (ms / reps / 1e3) / 1e9, e ? cudaGetErrorString(e) : "");
  return 0;
}
