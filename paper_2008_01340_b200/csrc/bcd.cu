// bcd.cu -- BCD NMF (Alg. 3, distBCDnmf; SURVEY s.8(f) f1) on
// the GPU, with the readings R22-R27 (DESIGN.md s.3): prox-linear block steps with the
// spectral norms of the r x r Grams as Lipschitz constants, column L1 normalisation of
// W with compensation into H, Nesterov extrapolation with delta-capped weights, and a
// correction that returns to the last accepted iterates when the objective rises.
// Kernels (any m x n, r <= 32; fp32 storage, fp64 for every sum and small matrix):
//   k_bcd_w      W = max(0, W_m - (W_m Q - P) / L_W), per row; column L1 partials
//   k_bcd_wnorm  W[:,k] /= c_k, W_prev[:,k] /= c_k (and G partials of the new W)
//   k_bcd_hnorm  H_m[k,:] *= c_k, H_prev[k,:] *= c_k
//   k_bcd_h      S = W^T X (fp32 per 128-row chunk, fp64 across), E = G H_m,
//                H = max(0, H_m - (E - S) / L_H), per column
//   k_bcd_obj    1/2 (||X||^2 - 2 <W, X H^T> + <W^T W, H H^T>) in fp64 (Gram identity)
//   k_bcd_extrap V_m = V + w (V - V_prev), V_prev = V
// The host drives the iteration (one 40-byte read-back per iteration for the
// correction / extrapolation decision, as Alg. 3 l.17 branches on the objective).
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ntt {

namespace {

constexpr int BROWS = 128;

template <int R>
__global__ void __launch_bounds__(BROWS)
k_bcd_w(const float* __restrict__ Wm, int64_t m, int r, const double* __restrict__ P, const double* __restrict__ Q,
        const double* __restrict__ LW, float* __restrict__ W, double* __restrict__ cpart) {
  __shared__ double Qs[R * R];
  __shared__ double cs[BROWS][R + 1];
  for (int t = threadIdx.x; t < R * R; t += blockDim.x) {
    const int k = t / R, l = t % R;
    Qs[t] = (k < r && l < r) ? Q[k * r + l] : 0.0;
  }
  __syncthreads();
  const double L = *LW;
  const int64_t i = (int64_t)blockIdx.x * BROWS + threadIdx.x;
  double w[R];
#pragma unroll
  for (int k = 0; k < R; ++k) w[k] = (i < m && k < r) ? (double)Wm[i * r + k] : 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    double v = 0.0;
    if (i < m && k < r) {
      double g = -P[i * r + k];
      for (int l = 0; l < r; ++l) g += w[l] * Qs[l * R + k];
      v = L > 0.0 ? fmax(0.0, w[k] - g / L) : w[k];
      const float vf = (float)v;
      W[i * r + k] = vf;
      v = (double)vf;
    }
    cs[threadIdx.x][k] = v;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < r; k += blockDim.x) {
    double s = 0.0;
    for (int q = 0; q < BROWS; ++q) s += cs[q][k];
    cpart[(int64_t)blockIdx.x * r + k] = s;
  }
}

// c = column sums (reduced); W, Wp columns /= c (c > 0); G partials of the normalised W
template <int R>
__global__ void __launch_bounds__(BROWS)
k_bcd_wnorm(float* __restrict__ W, float* __restrict__ Wp, int64_t m, int r, const double* __restrict__ c,
            double* __restrict__ Gpart) {
  __shared__ float Wn[BROWS][R + 1];
  const int64_t i = (int64_t)blockIdx.x * BROWS + threadIdx.x;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    float v = 0.0f;
    if (i < m && k < r) {
      const double ck = c ? c[k] : 0.0;  // c == nullptr: Gram partials only
      v = W[i * r + k];
      if (ck > 0.0) {
        v = (float)((double)v / ck);
        W[i * r + k] = v;
        Wp[i * r + k] = (float)((double)Wp[i * r + k] / ck);
      }
    }
    Wn[threadIdx.x][k] = v;
  }
  __syncthreads();
  const int rr = r * r;
  for (int t = threadIdx.x; t < rr; t += blockDim.x) {
    const int k = t / r, l = t % r;
    double s = 0.0;
    for (int q = 0; q < BROWS; ++q) s += (double)Wn[q][k] * (double)Wn[q][l];
    Gpart[(int64_t)blockIdx.x * rr + t] = s;
  }
}

__global__ void k_bcd_hnorm(float* __restrict__ Hm, float* __restrict__ Hp, int r, int64_t n,
                            const double* __restrict__ c) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)r * n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / n);
    const double ck = c[k];
    if (ck > 0.0) {
      Hm[e] = (float)((double)Hm[e] * ck);
      Hp[e] = (float)((double)Hp[e] * ck);
    }
  }
}

constexpr int BH_BN = 128;
constexpr int BH_MCH = 128;

template <int R>
__global__ void __launch_bounds__(BH_BN)
k_bcd_h(const float* __restrict__ X, int64_t ldx, int64_t m, int64_t n, const float* __restrict__ W, int r,
        const double* __restrict__ G, const double* __restrict__ LH, const float* __restrict__ Hm,
        float* __restrict__ H) {
  __shared__ float Ws[BH_MCH * R];
  __shared__ double Gs[R * R];
  for (int t = threadIdx.x; t < R * R; t += blockDim.x) {
    const int k = t / R, l = t % R;
    Gs[t] = (k < r && l < r) ? G[k * r + l] : 0.0;
  }
  const double L = *LH;
  const int64_t ntiles = (n + BH_BN - 1) / BH_BN;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t j = tile * BH_BN + threadIdx.x;
    const bool valid = j < n;
    double Sd[R];
#pragma unroll
    for (int k = 0; k < R; ++k) Sd[k] = 0.0;
    for (int64_t c0 = 0; c0 < m; c0 += BH_MCH) {
      const int rows = (int)min((int64_t)BH_MCH, m - c0);
      __syncthreads();
      for (int e = threadIdx.x; e < BH_MCH * R; e += blockDim.x) {
        const int ii = e / R, kk = e % R;
        Ws[e] = (ii < rows && kk < r) ? W[(c0 + ii) * r + kk] : 0.0f;
      }
      __syncthreads();
      float S[R];
#pragma unroll
      for (int k = 0; k < R; ++k) S[k] = 0.0f;
      if (valid)
        for (int ii = 0; ii < rows; ++ii) {
          const float x = X[(c0 + ii) * ldx + j];
#pragma unroll
          for (int k = 0; k < R; ++k) S[k] = fmaf(Ws[ii * R + k], x, S[k]);
        }
#pragma unroll
      for (int k = 0; k < R; ++k) Sd[k] += (double)S[k];
    }
    if (valid) {
      double hm[R];
#pragma unroll
      for (int k = 0; k < R; ++k) hm[k] = (k < r) ? (double)Hm[(int64_t)k * n + j] : 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (k >= r) continue;
        double e = -Sd[k];
#pragma unroll
        for (int l = 0; l < R; ++l) e += Gs[k * R + l] * hm[l];
        const double v = L > 0.0 ? fmax(0.0, hm[k] - e / L) : hm[k];
        H[(int64_t)k * n + j] = (float)v;
      }
    }
  }
}

// out[0] = 1/2 (xx - 2 <W, P> + <G, Q>) with W fp32 m x r, P fp64 m x r, G, Q fp64 r x r
__global__ void k_bcd_obj(double xx, const float* __restrict__ W, const double* __restrict__ P, int64_t m, int r,
                          const double* __restrict__ G, const double* __restrict__ Q, double* __restrict__ out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int64_t e = threadIdx.x; e < m * r; e += blockDim.x) s += (double)W[e] * P[e];
  double g = 0.0;
  for (int e = threadIdx.x; e < r * r; e += blockDim.x) g += G[e] * Q[e];
  double v = -2.0 * s + g;
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    out[0] = 0.5 * (xx + t);
  }
}

__global__ void k_bcd_extrap(float* __restrict__ V, float* __restrict__ Vm, float* __restrict__ Vp, int64_t cnt,
                             double w) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x) {
    const double v = V[e], vp = Vp[e];
    Vm[e] = (float)(v + w * (v - vp));
    Vp[e] = (float)v;
  }
}

__global__ void k_scale_copy(const float* __restrict__ src, float* __restrict__ a, float* __restrict__ b, int64_t cnt,
                             const double* __restrict__ num, const double* __restrict__ den) {
  const double s = sqrt(sqrt(*num)) / sqrt(*den);  // sqrt(||X||_F) / ||V||_F
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x) {
    const float v = (float)((double)src[e] * s);
    a[e] = v;
    b[e] = v;
  }
}

__global__ void k_sumsq(const float* __restrict__ v, int64_t rows, int64_t cols, int64_t ld, double* __restrict__ part) {
  double s = 0.0;
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x)
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
      const double x = v[i * ld + j];
      s += x * x;
    }
  s = warp_sum(s);
  __shared__ double red[32];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void k_copy_last(const double* __restrict__ eig, int N, double* __restrict__ out) {
  if (threadIdx.x == 0) out[0] = eig[N - 1];
}

int rcls_bcd(int r) { return r <= 4 ? 4 : r <= 8 ? 8 : r <= 16 ? 16 : 32; }

}  // namespace

int bcd_w_ctas(int64_t m) { return (int)((m + BROWS - 1) / BROWS); }

cudaError_t launch_bcd_w(const float* Wm, int64_t m, int r, const double* P, const double* Q, const double* LW,
                         float* W, double* cpart, cudaStream_t st) {
  const unsigned g = (unsigned)bcd_w_ctas(m);
  switch (rcls_bcd(r)) {
    case 4: k_bcd_w<4><<<g, BROWS, 0, st>>>(Wm, m, r, P, Q, LW, W, cpart); break;
    case 8: k_bcd_w<8><<<g, BROWS, 0, st>>>(Wm, m, r, P, Q, LW, W, cpart); break;
    case 16: k_bcd_w<16><<<g, BROWS, 0, st>>>(Wm, m, r, P, Q, LW, W, cpart); break;
    default: k_bcd_w<32><<<g, BROWS, 0, st>>>(Wm, m, r, P, Q, LW, W, cpart); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_bcd_wnorm(float* W, float* Wp, int64_t m, int r, const double* c, double* Gpart, cudaStream_t st) {
  const unsigned g = (unsigned)bcd_w_ctas(m);
  switch (rcls_bcd(r)) {
    case 4: k_bcd_wnorm<4><<<g, BROWS, 0, st>>>(W, Wp, m, r, c, Gpart); break;
    case 8: k_bcd_wnorm<8><<<g, BROWS, 0, st>>>(W, Wp, m, r, c, Gpart); break;
    case 16: k_bcd_wnorm<16><<<g, BROWS, 0, st>>>(W, Wp, m, r, c, Gpart); break;
    default: k_bcd_wnorm<32><<<g, BROWS, 0, st>>>(W, Wp, m, r, c, Gpart); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_bcd_hnorm(float* Hm, float* Hp, int r, int64_t n, const double* c, cudaStream_t st) {
  k_bcd_hnorm<<<1184, 256, 0, st>>>(Hm, Hp, r, n, c);
  return cudaGetLastError();
}

cudaError_t launch_bcd_h(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, int r, const double* G,
                         const double* LH, const float* Hm, float* H, int num_sms, cudaStream_t st) {
  int64_t g = (n + BH_BN - 1) / BH_BN;
  if (g > 8 * num_sms) g = 8 * num_sms;
  switch (rcls_bcd(r)) {
    case 4: k_bcd_h<4><<<(unsigned)g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, G, LH, Hm, H); break;
    case 8: k_bcd_h<8><<<(unsigned)g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, G, LH, Hm, H); break;
    case 16: k_bcd_h<16><<<(unsigned)g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, G, LH, Hm, H); break;
    default: k_bcd_h<32><<<(unsigned)g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, G, LH, Hm, H); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_bcd_obj(double xx, const float* W, const double* P, int64_t m, int r, const double* G,
                           const double* Q, double* out, cudaStream_t st) {
  k_bcd_obj<<<1, 1024, 0, st>>>(xx, W, P, m, r, G, Q, out);
  return cudaGetLastError();
}

cudaError_t launch_bcd_extrap(float* V, float* Vm, float* Vp, int64_t cnt, double w, cudaStream_t st) {
  k_bcd_extrap<<<1184, 256, 0, st>>>(V, Vm, Vp, cnt, w);
  return cudaGetLastError();
}

cudaError_t launch_scale_copy(const float* src, float* a, float* b, int64_t cnt, const double* num, const double* den,
                              cudaStream_t st) {
  k_scale_copy<<<1184, 256, 0, st>>>(src, a, b, cnt, num, den);
  return cudaGetLastError();
}

int sumsq_ctas() { return 1184; }

cudaError_t launch_sumsq(const float* v, int64_t rows, int64_t cols, int64_t ld, double* part, cudaStream_t st) {
  k_sumsq<<<1184, 256, 0, st>>>(v, rows, cols, ld, part);
  return cudaGetLastError();
}

cudaError_t launch_copy_last(const double* eig, int N, double* out, cudaStream_t st) {
  k_copy_last<<<1, 32, 0, st>>>(eig, N, out);
  return cudaGetLastError();
}

}  // namespace ntt
