// mu_generic.cu -- generic (any shape) MU-NMF building blocks for sm_100a.
//
// These kernels implement the W half-step and H half-step of the MU rule
// (include/ntt.h ntt_nmf_mu; readings R1-R4) for ANY m x n, including tall and
// square X (the "2-pass" form, SURVEY s.8(d)): an X H^T pass (Alg. 5 l.2,
// P:274) and Gram (Alg. 4), the W update, then a W^T X pass
// (Alg. 6 l.2) fused with the H update.  The H pass can also accumulate
// X H_new^T and H_new H_new^T for the next iteration (1-pass fusion) when m*r
// is small.  The fast short-wide path lives in mu_fused.cu.
//
// Accumulation: fp32 FMA within tiles, fp64 across tiles and CTAs (DESIGN.md
// s.5 "two-level sums"); cross-CTA partials are summed in a fixed order, so
// results are deterministic run to run.
#include "common.cuh"
#include "kernels.h"

namespace ntt {

// ---------------------------------------------------------------- RNG fill --
// 128-bit stores when p is 16-byte aligned (the first count & ~3 elements; the <= 3 left over
// by thread 0); element i is rng_uniform(key, off + i) either way
__global__ void k_fill_uniform(float* __restrict__ p, int64_t count, uint64_t key, int64_t off) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
    const int64_t n4 = count >> 2;
    for (int64_t q = i; q < n4; q += stride) {
      const uint64_t e = (uint64_t)(off + 4 * q);
      reinterpret_cast<float4*>(p)[q] =
          make_float4(rng_uniform(key, e), rng_uniform(key, e + 1), rng_uniform(key, e + 2), rng_uniform(key, e + 3));
    }
    if (i == 0)
      for (int64_t t = 4 * n4; t < count; ++t) p[t] = rng_uniform(key, (uint64_t)(off + t));
    return;
  }
  for (; i < count; i += stride) p[i] = rng_uniform(key, (uint64_t)(off + i));
}

cudaError_t launch_fill_uniform(float* p, int64_t count, uint64_t seed, uint64_t stream, int64_t off,
                                cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  k_fill_uniform<<<(unsigned)blocks, 256, 0, st>>>(p, count, rng_key(seed, stream), off);
  return cudaGetLastError();
}

// --------------------------------------------------------------- X H^T pass --
// CTA (cs, rb): rows [rb*32, rb*32+32), columns [cs*chunk, (cs+1)*chunk).
// Tiles of 32 rows x 64 columns of X and R x 64 of H are staged in smem; each
// thread owns (row, k) pairs and accumulates over the tile in fp32, folding
// into fp64 after every tile.
constexpr int XHT_MB = 32;
constexpr int XHT_TN = 64;
constexpr int XHT_THREADS = 256;

template <int R>
__global__ void __launch_bounds__(XHT_THREADS)
k_xht_partial(const float* __restrict__ X, int64_t ldx, int64_t m, int64_t n, const float* __restrict__ H,
              int64_t ldh, int r, int64_t chunk, double* __restrict__ Ppart) {
  __shared__ float Xs[XHT_MB][XHT_TN + 1];
  __shared__ float Hs[R][XHT_TN + 1];
  constexpr int NPAIR = XHT_MB * R;
  constexpr int PPT = (NPAIR + XHT_THREADS - 1) / XHT_THREADS;  // pairs per thread
  const int cs = blockIdx.x, rb = blockIdx.y;
  const int64_t i0 = (int64_t)rb * XHT_MB;
  const int64_t j0 = (int64_t)cs * chunk;
  const int64_t j1 = min(n, j0 + chunk);
  double acc[PPT];
#pragma unroll
  for (int q = 0; q < PPT; ++q) acc[q] = 0.0;

  for (int64_t jt = j0; jt < j1; jt += XHT_TN) {
    for (int e = threadIdx.x; e < XHT_MB * XHT_TN; e += XHT_THREADS) {
      int ii = e / XHT_TN, jj = e % XHT_TN;
      int64_t gi = i0 + ii, gj = jt + jj;
      Xs[ii][jj] = (gi < m && gj < j1) ? X[gi * ldx + gj] : 0.0f;
    }
    for (int e = threadIdx.x; e < R * XHT_TN; e += XHT_THREADS) {
      int kk = e / XHT_TN, jj = e % XHT_TN;
      int64_t gj = jt + jj;
      Hs[kk][jj] = (kk < r && gj < j1) ? H[(int64_t)kk * ldh + gj] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      int p = threadIdx.x + q * XHT_THREADS;
      if (p < NPAIR) {
        int ii = p / R, kk = p % R;
        float s = 0.0f;
#pragma unroll 8
        for (int jj = 0; jj < XHT_TN; ++jj) s = fmaf(Xs[ii][jj], Hs[kk][jj], s);
        acc[q] += (double)s;
      }
    }
    __syncthreads();
  }
  const int64_t mr = m * r;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    int p = threadIdx.x + q * XHT_THREADS;
    if (p < NPAIR) {
      int ii = p / R, kk = p % R;
      int64_t gi = i0 + ii;
      if (gi < m && kk < r) Ppart[(int64_t)cs * mr + gi * r + kk] = acc[q];
    }
  }
}

XhtPlan plan_xht(int64_t m, int64_t n, int num_sms) {
  XhtPlan pl;
  pl.nrb = (int)((m + XHT_MB - 1) / XHT_MB);
  int64_t want = (int64_t)num_sms * 4 / pl.nrb;
  if (want < 1) want = 1;
  int64_t tiles = (n + XHT_TN - 1) / XHT_TN;
  if (want > tiles) want = tiles;
  if (want > 4096) want = 4096;
  int64_t tpc = (tiles + want - 1) / want;  // tiles per chunk
  pl.chunk = tpc * XHT_TN;
  pl.ncs = (int)((n + pl.chunk - 1) / pl.chunk);
  return pl;
}

template <int R>
static cudaError_t xht_t(const float* X, int64_t ldx, int64_t m, int64_t n, const float* H, int64_t ldh, int r,
                         const XhtPlan& pl, double* Ppart, cudaStream_t st) {
  dim3 grid(pl.ncs, pl.nrb);
  k_xht_partial<R><<<grid, XHT_THREADS, 0, st>>>(X, ldx, m, n, H, ldh, r, pl.chunk, Ppart);
  return cudaGetLastError();
}

cudaError_t launch_xht_partial(const float* X, int64_t ldx, int64_t m, int64_t n, const float* H, int64_t ldh,
                               int r, const XhtPlan& pl, double* Ppart, cudaStream_t st) {
  if (r <= 2) return xht_t<2>(X, ldx, m, n, H, ldh, r, pl, Ppart, st);
  if (r <= 4) return xht_t<4>(X, ldx, m, n, H, ldh, r, pl, Ppart, st);
  if (r <= 8) return xht_t<8>(X, ldx, m, n, H, ldh, r, pl, Ppart, st);
  if (r <= 16) return xht_t<16>(X, ldx, m, n, H, ldh, r, pl, Ppart, st);
  if (r <= 32) return xht_t<32>(X, ldx, m, n, H, ldh, r, pl, Ppart, st);
  return xht_t<64>(X, ldx, m, n, H, ldh, r, pl, Ppart, st);
}

// ------------------------------------------------------------------ W update --
constexpr int wup_rows(int R) { return R <= 16 ? 128 : (R <= 32 ? 64 : 32); }

template <int R>
__global__ void __launch_bounds__(wup_rows(R))
k_wupdate(float* __restrict__ W, int64_t m, int r, const double* __restrict__ Ppart, int nP,
          const double* __restrict__ Qpart, int nQ, float eps, double* __restrict__ Gpart) {
  constexpr int WUP_ROWS = wup_rows(R);
  __shared__ double Qs[R * R];
  __shared__ float Wn[WUP_ROWS][R + 1];
  const int rr = r * r;
  for (int t = threadIdx.x; t < R * R; t += blockDim.x) {
    double s = 0.0;
    if (t < rr)
      for (int b = 0; b < nQ; ++b) s += Qpart[(int64_t)b * rr + t];
    Qs[t] = s;
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * WUP_ROWS + threadIdx.x;
  if (i < m) {
    const int64_t mr = m * r;
    double w[R];
#pragma unroll
    for (int k = 0; k < R; ++k) w[k] = (k < r) ? (double)W[i * r + k] : 0.0;
    for (int k = 0; k < r; ++k) {
      double p = 0.0;
      for (int b = 0; b < nP; ++b) p += Ppart[(int64_t)b * mr + i * r + k];
      double d = 0.0;
#pragma unroll
      for (int l = 0; l < R; ++l)
        if (l < r) d += w[l] * Qs[l * r + k];
      float wn = (float)mu_quot(w[k], p, d, (double)eps);
      Wn[threadIdx.x][k] = wn;
    }
    for (int k = 0; k < r; ++k) W[i * r + k] = Wn[threadIdx.x][k];
  } else {
    for (int k = 0; k < r; ++k) Wn[threadIdx.x][k] = 0.0f;
  }
  __syncthreads();
  // G partial over this CTA's rows (fixed order)
  for (int t = threadIdx.x; t < rr; t += blockDim.x) {
    int k = t / r, l = t % r;
    double s = 0.0;
    for (int q = 0; q < WUP_ROWS; ++q) s += (double)Wn[q][k] * (double)Wn[q][l];
    Gpart[(int64_t)blockIdx.x * rr + t] = s;
  }
}

static int wup_rows_rt(int r) { return r <= 2 ? wup_rows(2) : r <= 4 ? wup_rows(4) : r <= 8 ? wup_rows(8) : r <= 16 ? wup_rows(16) : r <= 32 ? wup_rows(32) : wup_rows(64); }
int wupdate_ctas(int64_t m, int r) { return (int)((m + wup_rows_rt(r) - 1) / wup_rows_rt(r)); }

cudaError_t launch_wupdate(float* W, int64_t m, int r, const double* Ppart, int nP, const double* Qpart, int nQ,
                           float eps, double* Gpart, cudaStream_t st) {
  int grid = wupdate_ctas(m, r);
#define WUP(RR) k_wupdate<RR><<<grid, wup_rows(RR), 0, st>>>(W, m, r, Ppart, nP, Qpart, nQ, eps, Gpart)
  if (r <= 2) WUP(2);
  else if (r <= 4) WUP(4);
  else if (r <= 8) WUP(8);
  else if (r <= 16) WUP(16);
  else if (r <= 32) WUP(32);
  else WUP(64);
#undef WUP
  return cudaGetLastError();
}

// -------------------------------------------------------------------- H pass --
// Persistent CTAs over column tiles of HP_BN columns; one thread per column.
constexpr int HP_BN = 128;
constexpr int HP_MCH = 128;  // W rows staged per chunk

template <int R, bool ACC>
__global__ void __launch_bounds__(HP_BN)
k_hpass(const float* __restrict__ X, int64_t ldx, int64_t m, int64_t n, const float* __restrict__ W, int r,
        const double* __restrict__ Gpart, int nG, float eps, float* __restrict__ H, double* __restrict__ Ppart,
        double* __restrict__ Qpart) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* Gs = reinterpret_cast<float*>(smem_raw);                 // R*R
  float* Ws = Gs + R * R;                                          // HP_MCH*R
  float* Hs = Ws + HP_MCH * R;                                     // R*HP_BN (ACC only)
  double* Pacc = reinterpret_cast<double*>(Hs + (ACC ? R * HP_BN : 0));  // m*r (ACC)
  double* Qacc = Pacc + (ACC ? m * r : 0);                         // r*r (ACC)
  const int rr = r * r;
  for (int t = threadIdx.x; t < R * R; t += blockDim.x) {
    int k = t / R, l = t % R;
    double s = 0.0;
    if (k < r && l < r)
      for (int b = 0; b < nG; ++b) s += Gpart[(int64_t)b * rr + k * r + l];
    Gs[t] = (float)s;
  }
  if (ACC) {
    for (int64_t t = threadIdx.x; t < m * r; t += blockDim.x) Pacc[t] = 0.0;
    for (int t = threadIdx.x; t < rr; t += blockDim.x) Qacc[t] = 0.0;
  }
  __syncthreads();
  const int64_t ntiles = (n + HP_BN - 1) / HP_BN;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t j = tile * HP_BN + threadIdx.x;
    const bool valid = j < n;
    double Sd[R];
#pragma unroll
    for (int k = 0; k < R; ++k) Sd[k] = 0.0;
    for (int64_t c0 = 0; c0 < m; c0 += HP_MCH) {
      const int rows = (int)min((int64_t)HP_MCH, m - c0);
      __syncthreads();
      for (int e = threadIdx.x; e < HP_MCH * R; e += blockDim.x) {
        int ii = e / R, kk = e % R;
        Ws[e] = (ii < rows && kk < r) ? W[(c0 + ii) * r + kk] : 0.0f;
      }
      __syncthreads();
      float S[R];
#pragma unroll
      for (int k = 0; k < R; ++k) S[k] = 0.0f;
      if (valid) {
        for (int ii = 0; ii < rows; ++ii) {
          float x = X[(c0 + ii) * ldx + j];
#pragma unroll
          for (int k = 0; k < R; ++k) S[k] = fmaf(Ws[ii * R + k], x, S[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < R; ++k) Sd[k] += (double)S[k];
    }
    float hn[R];
    if (valid) {
      float h[R];
#pragma unroll
      for (int k = 0; k < R; ++k) h[k] = (k < r) ? H[(int64_t)k * n + j] : 0.0f;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        float e = 0.0f;
#pragma unroll
        for (int l = 0; l < R; ++l) e = fmaf(Gs[k * R + l], h[l], e);
        hn[k] = (k < r) ? mu_quot(h[k], (float)Sd[k], e, eps) : 0.0f;
      }
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (k < r) H[(int64_t)k * n + j] = hn[k];
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) hn[k] = 0.0f;
    }
    if (ACC) {
      __syncthreads();
#pragma unroll
      for (int k = 0; k < R; ++k) Hs[k * HP_BN + threadIdx.x] = hn[k];
      __syncthreads();
      const int64_t jb = tile * HP_BN;
      const int cols = (int)min((int64_t)HP_BN, n - jb);
      for (int64_t p = threadIdx.x; p < m * r; p += blockDim.x) {
        int64_t ii = p / r;
        int kk = (int)(p % r);
        const float* xr = X + ii * ldx + jb;
        float s = 0.0f;
        for (int c = 0; c < cols; ++c) s = fmaf(xr[c], Hs[kk * HP_BN + c], s);
        Pacc[p] += (double)s;
      }
      for (int p = threadIdx.x; p < rr; p += blockDim.x) {
        int k = p / r, l = p % r;
        float s = 0.0f;
        for (int c = 0; c < cols; ++c) s = fmaf(Hs[k * HP_BN + c], Hs[l * HP_BN + c], s);
        Qacc[p] += (double)s;
      }
    }
  }
  if (ACC) {
    __syncthreads();
    for (int64_t p = threadIdx.x; p < m * r; p += blockDim.x) Ppart[(int64_t)blockIdx.x * m * r + p] = Pacc[p];
    for (int p = threadIdx.x; p < rr; p += blockDim.x) Qpart[(int64_t)blockIdx.x * rr + p] = Qacc[p];
  }
}

int hpass_ctas(int64_t m, int64_t n, int r, bool acc, int num_sms) {
  int64_t ntiles = (n + HP_BN - 1) / HP_BN;
  int64_t g = (int64_t)num_sms * (acc ? 4 : 8);
  if (g > ntiles) g = ntiles;
  if (g < 1) g = 1;
  return (int)g;
}

template <int R>
static cudaError_t hpass_t(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, int r,
                           const double* Gpart, int nG, float eps, float* H, int grid, double* Ppart,
                           double* Qpart, cudaStream_t st) {
  size_t base = sizeof(float) * (R * R + HP_MCH * R);
  if (Ppart) {
    size_t sm = base + sizeof(float) * R * HP_BN + sizeof(double) * (size_t)(m * r + r * r);
    sm = (sm + 15) & ~(size_t)15;
    cudaError_t e = smem_optin((const void*)(k_hpass<R, true>), sm);
    if (e != cudaSuccess) return e;
    k_hpass<R, true><<<grid, HP_BN, sm, st>>>(X, ldx, m, n, W, r, Gpart, nG, eps, H, Ppart, Qpart);
  } else {
    k_hpass<R, false><<<grid, HP_BN, base, st>>>(X, ldx, m, n, W, r, Gpart, nG, eps, H, nullptr, nullptr);
  }
  return cudaGetLastError();
}

// Split-K H pass for few column tiles and many rows (e.g. the 500 GB tensor's step 3, 15360 x 64,
// r 40: one 128-column tile left one CTA walking all rows).  k_hpass_sk: CTA (tile, split) sums
// S = W^T X over its rows (fp32 per HP_MCH-row chunk, fp64 across, as k_hpass) into
// Spart[split][j][R]; k_hpass_fin: CTA of 256 threads = HF_C columns x R ranks sums the splits in
// order (fp64), then thread (column, rank) applies the MU H update.
template <int R>
__global__ void __launch_bounds__(HP_BN)
k_hpass_sk(const float* __restrict__ X, int64_t ldx, int64_t m, int64_t n, const float* __restrict__ W, int r, int ks,
           double* __restrict__ Spart) {
  __shared__ float Ws[HP_MCH * R];
  const int64_t tile = blockIdx.x, k = blockIdx.y;
  const int64_t i0 = m * k / ks, i1 = m * (k + 1) / ks;
  const int64_t j = tile * HP_BN + threadIdx.x;
  const bool valid = j < n;
  double Sd[R];
#pragma unroll
  for (int q = 0; q < R; ++q) Sd[q] = 0.0;
  for (int64_t c0 = i0; c0 < i1; c0 += HP_MCH) {
    const int rows = (int)min((int64_t)HP_MCH, i1 - c0);
    __syncthreads();
    for (int e = threadIdx.x; e < HP_MCH * R; e += blockDim.x) {
      const int ii = e / R, kk = e % R;
      Ws[e] = (ii < rows && kk < r) ? W[(c0 + ii) * r + kk] : 0.0f;
    }
    __syncthreads();
    float S[R];
#pragma unroll
    for (int q = 0; q < R; ++q) S[q] = 0.0f;
    if (valid)
      for (int ii = 0; ii < rows; ++ii) {
        const float x = X[(c0 + ii) * ldx + j];
#pragma unroll
        for (int q = 0; q < R; ++q) S[q] = fmaf(Ws[ii * R + q], x, S[q]);
      }
#pragma unroll
    for (int q = 0; q < R; ++q) Sd[q] += (double)S[q];
  }
  if (valid) {
    double* dst = Spart + ((int64_t)k * n + j) * R;
#pragma unroll
    for (int q = 0; q < R; ++q) dst[q] = Sd[q];
  }
}

constexpr int HF_T = 256;
template <int R>
__global__ void __launch_bounds__(HF_T)
k_hpass_fin(int64_t n, int r, int ks, const double* __restrict__ Spart, const double* __restrict__ Gred,
            float eps, float* __restrict__ H) {
  constexpr int C = HF_T / R;  // columns per CTA
  __shared__ float Gs[R * R];
  __shared__ float Hc[C][R];
  for (int t = threadIdx.x; t < R * R; t += HF_T) {  // G already summed over its partials (r x r)
    const int a = t / R, b = t % R;
    Gs[t] = (a < r && b < r) ? (float)Gred[a * r + b] : 0.0f;
  }
  const int c = threadIdx.x / R, kk = threadIdx.x % R;
  const int64_t j = (int64_t)blockIdx.x * C + c;
  const bool valid = j < n && kk < r;
  Hc[c][kk] = valid ? H[(int64_t)kk * n + j] : 0.0f;
  double sd = 0.0;
  if (valid) {
    const double* src = Spart + j * R + kk;
    const int64_t stride = n * R;
    int q = 0;
    for (; q + 8 <= ks; q += 8) {  // 8 loads in flight, summed in split order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(src + (int64_t)(q + u) * stride);
#pragma unroll
      for (int u = 0; u < 8; ++u) sd += v[u];
    }
    for (; q < ks; ++q) sd += __ldcg(src + (int64_t)q * stride);
  }
  __syncthreads();
  if (valid) {
    float e = 0.0f;
#pragma unroll
    for (int l = 0; l < R; ++l) e = fmaf(Gs[kk * R + l], Hc[c][l], e);
    H[(int64_t)kk * n + j] = mu_quot(Hc[c][kk], (float)sd, e, eps);
  }
}

// split count of the split-K H pass (0 = the per-tile kernel): few column tiles, many rows
int hpass_splits(int64_t m, int64_t n, int num_sms) {
  const int64_t ntiles = (n + HP_BN - 1) / HP_BN;
  if (ntiles * 4 > num_sms || m < 1024) return 0;
  int64_t ks = std::min<int64_t>(m / 64, (2 * num_sms + ntiles - 1) / ntiles);
  return ks >= 2 ? (int)ks : 0;
}

cudaError_t launch_hpass_sk(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, int r,
                            const double* Gpart, int nG, float eps, float* H, int ks, double* Spart, double* Gred,
                            cudaStream_t st) {
  const int64_t ntiles = (n + HP_BN - 1) / HP_BN;
  cudaError_t e0 = launch_sum_partials(Gpart, nG, (int64_t)r * r, Gred, st);  // fixed order
  if (e0 != cudaSuccess) return e0;
#define HSK(RR)                                                                                         \
  do {                                                                                                  \
    k_hpass_sk<RR><<<dim3((unsigned)ntiles, (unsigned)ks), HP_BN, 0, st>>>(X, ldx, m, n, W, r, ks, Spart); \
    k_hpass_fin<RR><<<(unsigned)((n + HF_T / RR - 1) / (HF_T / RR)), HF_T, 0, st>>>(n, r, ks, Spart, Gred, eps, \
                                                                                     H);                \
  } while (0)
  if (r <= 2) HSK(2);
  else if (r <= 4) HSK(4);
  else if (r <= 8) HSK(8);
  else if (r <= 16) HSK(16);
  else if (r <= 32) HSK(32);
  else HSK(64);
#undef HSK
  return cudaGetLastError();
}

cudaError_t launch_hpass(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, int r,
                         const double* Gpart, int nG, float eps, float* H, int grid, double* Ppart, double* Qpart,
                         cudaStream_t st) {
  if (r <= 2) return hpass_t<2>(X, ldx, m, n, W, r, Gpart, nG, eps, H, grid, Ppart, Qpart, st);
  if (r <= 4) return hpass_t<4>(X, ldx, m, n, W, r, Gpart, nG, eps, H, grid, Ppart, Qpart, st);
  if (r <= 8) return hpass_t<8>(X, ldx, m, n, W, r, Gpart, nG, eps, H, grid, Ppart, Qpart, st);
  if (r <= 16) return hpass_t<16>(X, ldx, m, n, W, r, Gpart, nG, eps, H, grid, Ppart, Qpart, st);
  if (r <= 32) return hpass_t<32>(X, ldx, m, n, W, r, Gpart, nG, eps, H, grid, Ppart, Qpart, st);
  return hpass_t<64>(X, ldx, m, n, W, r, Gpart, nG, eps, H, grid, Ppart, Qpart, st);
}

// ----------------------------------------------------------------- objective --
constexpr int OBJ_THREADS = 256;

__global__ void __launch_bounds__(OBJ_THREADS)
k_objective(const float* __restrict__ X, int64_t ldx, int64_t m, int64_t n, const float* __restrict__ W,
            const float* __restrict__ H, int r, double* __restrict__ part) {
  __shared__ double red[OBJ_THREADS / 32];
  double acc = 0.0;
  for (int64_t j = (int64_t)blockIdx.x * OBJ_THREADS + threadIdx.x; j < n; j += (int64_t)gridDim.x * OBJ_THREADS) {
    for (int64_t i = 0; i < m; ++i) {
      double wh = 0.0;
      for (int k = 0; k < r; ++k) wh += (double)W[i * r + k] * (double)H[(int64_t)k * n + j];
      double e = (double)X[i * ldx + j] - wh;
      acc += e * e;
    }
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < OBJ_THREADS / 32; ++w) s += red[w];
    part[blockIdx.x] = s;
  }
}

int objective_ctas(int64_t n) {
  int64_t g = (n + OBJ_THREADS - 1) / OBJ_THREADS;
  return (int)(g > 1184 ? 1184 : g);
}

cudaError_t launch_objective(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, const float* H,
                             int r, double* part, cudaStream_t st) {
  k_objective<<<objective_ctas(n), OBJ_THREADS, 0, st>>>(X, ldx, m, n, W, H, r, part);
  return cudaGetLastError();
}

}  // namespace ntt

namespace ntt {

__global__ void k_sum_partials(const double* __restrict__ part, int nparts, int64_t len, double* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < len; t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += part[(int64_t)b * len + t];
    out[t] = s;
  }
}

// few outputs, many partials: one warp per output, lanes take every 32nd partial, then a fixed
// shuffle tree (deterministic; avoids a serial chain of nparts dependent-latency loads)
__global__ void k_sum_partials_warp(const double* __restrict__ part, int nparts, int64_t len, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (t >= len) return;
  double s = 0.0;
  for (int b = threadIdx.x & 31; b < nparts; b += 32) s += part[(int64_t)b * len + t];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) out[t] = s;
}

cudaError_t launch_sum_partials(const double* part, int nparts, int64_t len, double* out, cudaStream_t st) {
  if (nparts >= 8 && len <= 4096) {
    k_sum_partials_warp<<<(unsigned)((len + 7) / 8), 256, 0, st>>>(part, nparts, len, out);
    return cudaGetLastError();
  }
  int64_t g = (len + 255) / 256;
  if (g > 1184) g = 1184;
  if (g < 1) g = 1;
  k_sum_partials<<<(unsigned)g, 256, 0, st>>>(part, nparts, len, out);
  return cudaGetLastError();
}

__global__ void k_fill_uniform_cols(float* __restrict__ H, int r, int64_t nloc, int64_t b, int64_t nd, int64_t off,
                                    int64_t nglob, uint64_t key) {
  const int64_t total = (int64_t)r * nloc;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = t / nloc, c = t - k * nloc;
    int64_t cg = (c / b) * nd + off + (c % b);
    H[t] = rng_uniform(key, (uint64_t)(k * nglob + cg));
  }
}

cudaError_t launch_fill_uniform_cols(float* H, int r, int64_t nloc, int64_t b, int64_t nd, int64_t off, int64_t nglob,
                                     uint64_t seed, uint64_t stream, cudaStream_t st) {
  int64_t total = (int64_t)r * nloc;
  int64_t g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  if (g < 1) g = 1;
  k_fill_uniform_cols<<<(unsigned)g, 256, 0, st>>>(H, r, nloc, b, nd, off, nglob, rng_key(seed, stream));
  return cudaGetLastError();
}

__global__ void k_gather_last_core(const float* __restrict__ gath, int64_t r, int64_t nd, int nranks,
                                   float* __restrict__ core) {
  const int64_t total = r * nd;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t k = t / nd, i = t - k * nd;
    // rank g owning column i: b_g = floor(g nd / p); find g with b_g <= i < b_{g+1}
    int g = (int)(((i + 1) * nranks - 1) / nd);
    while (g > 0 && nd * g / nranks > i) --g;
    while (g + 1 < nranks && nd * (g + 1) / nranks <= i) ++g;
    int64_t og = nd * g / nranks, bg = nd * (g + 1) / nranks - og;
    core[t] = gath[r * og + k * bg + (i - og)];
  }
}

cudaError_t launch_gather_last_core(const float* gath, int64_t r, int64_t nd, int nranks, float* core, cudaStream_t st) {
  int64_t g = (r * nd + 255) / 256;
  if (g < 1) g = 1;
  k_gather_last_core<<<(unsigned)g, 256, 0, st>>>(gath, r, nd, nranks, core);
  return cudaGetLastError();
}

}  // namespace ntt

namespace ntt {
namespace {
// validation (ntt_set_validation): count the entries of a rows x cols matrix (row stride ld)
// that are not >= 0 -- negative values and NaNs (SPEC's NonnegativityError)
__global__ void k_count_not_nonneg(const float* __restrict__ v, int64_t rows, int64_t cols, int64_t ld,
                                   unsigned long long* __restrict__ bad) {
  unsigned long long c = 0;
  const int64_t total = rows * cols;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / cols, j = e - i * cols;
    c += !(__ldg(v + i * ld + j) >= 0.0f);
  }
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(bad, c);
}
}  // namespace

cudaError_t launch_count_not_nonneg(const float* v, int64_t rows, int64_t cols, int64_t ld, unsigned long long* bad,
                                    int num_sms, cudaStream_t st) {
  cudaMemsetAsync(bad, 0, sizeof(unsigned long long), st);
  const int64_t total = rows * cols;
  int64_t blocks = std::min<int64_t>((total + 255) / 256, (int64_t)num_sms * 8);
  if (blocks < 1) blocks = 1;
  k_count_not_nonneg<<<(unsigned)blocks, 256, 0, st>>>(v, rows, cols, ld, bad);
  return cudaGetLastError();
}
}  // namespace ntt
