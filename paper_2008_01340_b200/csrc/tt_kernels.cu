// tt_kernels.cu -- tensor-train contraction (Eq. 1), relative error
// (Eq. 3) and synthetic-tensor generation for sm_100a.
//
// The train is split at a middle bond k:  A~[a, b] = sum_q L_k[a, q] R_k[q, b]
// with L_k = G_1 o ... o G_k  (N_L x r_k) and R_k = G_{k+1} o ... o G_d
// (r_k x N_R).  L and R are built by small contraction kernels; the streaming
// kernel then forms every element with r_k FMAs while it streams the reference
// tensor once (the HBM-bound part), accumulating ||ref - A~||^2 and ||ref||^2
// with fp32 per element and fp64 per-thread sums.
#include "common.cuh"
#include "kernels.h"

namespace ntt {

__global__ void k_contract_left(const float* __restrict__ L, int64_t N, int rp, const float* __restrict__ G,
                                int64_t nl, int rl, float* __restrict__ out) {
  const int64_t total = N * nl * rl;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t c = t % rl;
    int64_t i = (t / rl) % nl;
    int64_t a = t / (rl * nl);
    float s = 0.0f;
    for (int k = 0; k < rp; ++k) s = fmaf(L[a * rp + k], G[((int64_t)k * nl + i) * rl + c], s);
    out[t] = s;
  }
}

__global__ void k_contract_right(const float* __restrict__ G, int rp, int64_t nl, int rl, const float* __restrict__ R,
                                 int64_t NR, float* __restrict__ out) {
  const int64_t total = (int64_t)rp * nl * NR;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = t % NR;
    int64_t i = (t / NR) % nl;
    int64_t k = t / (NR * nl);
    float s = 0.0f;
    for (int c = 0; c < rl; ++c) s = fmaf(G[(k * nl + i) * rl + c], R[(int64_t)c * NR + b], s);
    out[t] = s;
  }
}

static unsigned grid_for(int64_t total) {
  int64_t b = (total + 255) / 256;
  return (unsigned)(b > 148 * 16 ? 148 * 16 : (b < 1 ? 1 : b));
}

cudaError_t launch_contract_left(const float* L, int64_t N, int rp, const float* G, int64_t nl, int rl, float* out,
                                 cudaStream_t st) {
  k_contract_left<<<grid_for(N * nl * rl), 256, 0, st>>>(L, N, rp, G, nl, rl, out);
  return cudaGetLastError();
}

cudaError_t launch_contract_right(const float* G, int rp, int64_t nl, int rl, const float* R, int64_t NR, float* out,
                                  cudaStream_t st) {
  k_contract_right<<<grid_for((int64_t)rp * nl * NR), 256, 0, st>>>(G, rp, nl, rl, R, NR, out);
  return cudaGetLastError();
}

// Streaming kernel: CTA handles rows a of A~ (grid-stride), threads over b.
constexpr int TS_THREADS = 256;

template <int RK>
__global__ void __launch_bounds__(TS_THREADS)
k_tt_stream(const float* __restrict__ L, const float* __restrict__ R, int64_t NL, int64_t NR, int rk,
            float* __restrict__ out, float noise_amp, uint64_t noise_key, const float* __restrict__ ref,
            double* __restrict__ err_part) {
  __shared__ double red[2][TS_THREADS / 32];
  double num = 0.0, den = 0.0;
  const int64_t total = NL * NR;
  for (int64_t t = (int64_t)blockIdx.x * TS_THREADS + threadIdx.x; t < total; t += (int64_t)gridDim.x * TS_THREADS) {
    const int64_t a = t / NR, b = t - a * NR;
    float s = 0.0f;
#pragma unroll
    for (int q = 0; q < RK; ++q)
      if (q < rk) s = fmaf(L[a * rk + q], R[(int64_t)q * NR + b], s);
    if (out) {
      float v = s;
      if (noise_amp != 0.0f) v = __fadd_rn(v, __fmul_rn(noise_amp, rng_uniform(noise_key, (uint64_t)t)));
      out[t] = v;
    }
    if (ref) {
      float x = ref[t];
      double e = (double)x - (double)s;
      num += e * e;
      den += (double)x * (double)x;
    }
  }
  if (ref) {
    num = warp_sum(num);
    den = warp_sum(den);
    if ((threadIdx.x & 31) == 0) {
      red[0][threadIdx.x >> 5] = num;
      red[1][threadIdx.x >> 5] = den;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double sn = 0.0, sd = 0.0;
      for (int w = 0; w < TS_THREADS / 32; ++w) {
        sn += red[0][w];
        sd += red[1][w];
      }
      err_part[2 * blockIdx.x] = sn;
      err_part[2 * blockIdx.x + 1] = sd;
    }
  }
}

int stream_ctas(int64_t NL, int64_t NR, int num_sms) {
  int64_t total = NL * NR;
  int64_t g = (total + TS_THREADS - 1) / TS_THREADS;
  int64_t cap = (int64_t)num_sms * 8;
  return (int)(g > cap ? cap : (g < 1 ? 1 : g));
}

cudaError_t launch_tt_stream(const float* L, const float* R, int64_t NL, int64_t NR, int rk, float* out,
                             float noise_amp, uint64_t noise_key, const float* ref, double* err_part, int grid,
                             cudaStream_t st) {
#define TS(K) k_tt_stream<K><<<grid, TS_THREADS, 0, st>>>(L, R, NL, NR, rk, out, noise_amp, noise_key, ref, err_part)
  if (rk <= 1) TS(1);
  else if (rk <= 2) TS(2);
  else if (rk <= 4) TS(4);
  else if (rk <= 8) TS(8);
  else if (rk <= 16) TS(16);
  else if (rk <= 32) TS(32);
  else TS(64);
#undef TS
  return cudaGetLastError();
}

}  // namespace ntt
