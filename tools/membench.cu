// membench.cu -- HBM rate of a multi-row streaming pattern (tools only):
// out[k][j] = in_h[k][j] * sum_i x[i][j] for i < RX rows of X and k < RH rows of H (read X, read H,
// write H), rows of pitch `pitch` floats.  Prints GB/s (algorithmic bytes / CUDA-event time).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/membench tools/membench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void k_rows(const float* __restrict__ X, int rx, float* __restrict__ H, int rh, long long n, long long pitch) {
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < n / 4; j += (long long)gridDim.x * blockDim.x) {
    float4 s = make_float4(0, 0, 0, 0);
    for (int i = 0; i < rx; ++i) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(X + i * pitch) + j);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    for (int k = 0; k < rh; ++k) {
      float4* p = reinterpret_cast<float4*>(H + k * pitch) + j;
      float4 h = *p;
      h.x = h.x * s.x / (s.x + 1.0f); h.y = h.y * s.y / (s.y + 1.0f);
      h.z = h.z * s.z / (s.z + 1.0f); h.w = h.w * s.w / (s.w + 1.0f);
      *p = h;
    }
  }
}

int main(int argc, char** argv) {
  const long long n = argc > 1 ? atoll(argv[1]) : 10077696;
  const long long pitch = argc > 2 ? atoll(argv[2]) : n;
  const int rx = argc > 3 ? atoi(argv[3]) : 6, rh = argc > 4 ? atoi(argv[4]) : 5;
  const int bps = argc > 5 ? atoi(argv[5]) : 8, thr = argc > 6 ? atoi(argv[6]) : 256;
  float *X, *H;
  cudaMalloc(&X, sizeof(float) * pitch * rx);
  cudaMalloc(&H, sizeof(float) * pitch * rh);
  {  // non-trivial data (some memory systems treat zero pages specially)
    float* hb = (float*)malloc(sizeof(float) * pitch);
    for (long long q = 0; q < pitch; ++q) hb[q] = 1.0f + (float)((q * 2654435761ull) % 1000) * 1e-3f;
    for (int i = 0; i < rx; ++i) cudaMemcpy(X + i * pitch, hb, sizeof(float) * pitch, cudaMemcpyHostToDevice);
    for (int k = 0; k < rh; ++k) cudaMemcpy(H + k * pitch, hb, sizeof(float) * pitch, cudaMemcpyHostToDevice);
    free(hb);
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) k_rows<<<sms * bps, thr>>>(X, rx, H, rh, n, pitch);
  cudaEventRecord(a);
  const int reps = 20;
  for (int it = 0; it < reps; ++it) k_rows<<<sms * bps, thr>>>(X, rx, H, rh, n, pitch);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = 4.0 * n * (rx + 2.0 * rh);
  printf("n=%lld pitch=%lld rx=%d rh=%d grid=%dx%d : %.1f GB/s (%.3f ms/pass)\n", n, pitch, rx, rh, sms * bps, thr, bytes / (ms / reps / 1e3) / 1e9,
         ms / reps);
  return 0;
}
