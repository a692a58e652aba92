// Probe: persist_step's W update (m x r, fp64) in isolation, one CTA, clock64.  Not product.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double mu_quot(double w, double num, double den, double eps) {
  return __ddiv_rn(__dmul_rn(w, num), __dadd_rn(den, eps));
}
template <int MODE>
__global__ void k(const double* __restrict__ srcv, float* Wout, int m, int r, float eps, long long* cyc) {
  __shared__ double scr[4096];
  __shared__ float Ws[256 * 8];
  const int T = blockDim.x, tid = threadIdx.x;
  const int L = m * r + r * r;
  for (int e = tid; e < m * 8; e += T) Ws[e] = 0.5f + (e % 7) * 0.1f;
  for (int e = tid; e < L; e += T) scr[e] = srcv[e];
  __syncthreads();
  double* P = scr;
  double* Q = scr + m * r;
  float* Wn = reinterpret_cast<float*>(scr + L + 16);
  long long t0 = clock64();
  if (MODE == 3) {
    for (int i = tid; i < m; i += T) {
      double w[8];
#pragma unroll
      for (int l = 0; l < 8; ++l) w[l] = (double)Ws[i * 8 + l];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int l = 0; l < 8; l += 2) {
          d0 += w[l] * Q[l * 8 + k];
          d1 += w[l + 1] * Q[(l + 1) * 8 + k];
        }
        Wn[i * 8 + k] = (float)mu_quot(w[k], P[i * 8 + k], d0 + d1, (double)eps);
      }
    }
  } else
  for (int e0 = tid; e0 < m * 8; e0 += 4 * T) {
    double d[4], wv[4], pv[4];
    int ii[4], kk[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * T;
      ii[u] = e >> 3;
      kk[u] = e & 7;
      const bool ok = e < m * 8 && kk[u] < r;
      wv[u] = ok ? (double)Ws[ii[u] * 8 + kk[u]] : 0.0;
      pv[u] = ok ? P[ii[u] * r + kk[u]] : 0.0;
      d[u] = 0.0;
    }
    for (int l = 0; l < r; ++l) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * T;
        if (e < m * 8 && kk[u] < r) d[u] += (double)Ws[ii[u] * 8 + l] * Q[l * r + kk[u]];
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = e0 + u * T;
      if (e < m * 8) Wn[e] = kk[u] < r ? (MODE == 0 ? (float)mu_quot(wv[u], pv[u], d[u], (double)eps)
                                          : MODE == 1 ? (float)(wv[u] * pv[u] * d[u])
                                                      : __fdiv_rn((float)(wv[u] * pv[u]), (float)(d[u] + eps))) : 0.0f;
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (tid == 0) cyc[0] = t1 - t0;
  for (int e = tid; e < m * 8; e += T) Wout[e] = Wn[e];
}
int main() {
  double* s; float* w; long long* c;
  cudaMalloc(&s, 8 * 4096); cudaMalloc(&w, 4 * 4096); cudaMallocManaged(&c, 64);
  { double hs[4096]; for (int i = 0; i < 4096; ++i) hs[i] = 0.5 + (i % 13) * 0.01; cudaMemcpy(s, hs, sizeof hs, cudaMemcpyHostToDevice); }
  for (int T : {160, 288})
    for (int m : {30, 256}) {
      long long r3[3];
      k<0><<<1, T>>>(s, w, m, 8, 1e-16f, c); cudaDeviceSynchronize();
      k<0><<<1, T>>>(s, w, m, 8, 1e-16f, c); cudaDeviceSynchronize(); r3[0] = c[0];
      k<1><<<1, T>>>(s, w, m, 8, 1e-16f, c); cudaDeviceSynchronize();
      k<1><<<1, T>>>(s, w, m, 8, 1e-16f, c); cudaDeviceSynchronize(); r3[1] = c[0];
      k<2><<<1, T>>>(s, w, m, 8, 1e-16f, c); cudaDeviceSynchronize();
      k<2><<<1, T>>>(s, w, m, 8, 1e-16f, c); cudaDeviceSynchronize(); r3[2] = c[0];
      k<3><<<1, T>>>(s, w, m, 8, 1e-16f, c); cudaDeviceSynchronize();
      k<3><<<1, T>>>(s, w, m, 8, 1e-16f, c); cudaDeviceSynchronize();
      printf("T=%d m=%d: W update cycles: fp64 div %lld, no div %lld, fp32 div %lld, row-per-thread %lld\n", T, m, r3[0], r3[1], r3[2], c[0]);
    }
  return 0;
}
