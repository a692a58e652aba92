// bcd.cu -- BCD NMF (Alg. 3, distBCDnmf; SURVEY s.8(f) f1) on
// the GPU, with the readings R22-R27 (DESIGN.md s.3): prox-linear block steps with the
// spectral norms of the r x r Grams as Lipschitz constants, column L1 normalisation of
// W with compensation into H, Nesterov extrapolation with delta-capped weights, and a
// correction that returns to the last accepted iterates when the objective rises.
// Kernels (any m x n, r <= 32; fp32 storage, fp64 for every sum and small matrix):
//   k_bcd_w      W = max(0, W_m - (W_m Q - P) / L_W), per row; column L1 partials
//   k_bcd_wnorm  W[:,k] /= c_k, W_prev[:,k] /= c_k (and G partials of the new W)
//   k_bcd_hscale the same for H through row-scale vectors of H_m and H_prev (no H traffic)
//   k_bcd_spart  split-K partials of S = W^T X (FFMA path; the tensor-core path
//                produces the same [split][j][k] layout with k_skinny_tc16<R, 1>)
//   k_bcd_hup    S = sum of the partials, E = G H_m, H = max(0, H_m - (E - S) / L_H)
//   k_bcd_psum_dot  P = X H^T from its split partials, with per-CTA partials of <W, P>
//   k_spec_norm  ||M||_2 of an r x r Gram (repeated squaring + Rayleigh quotient)
//   k_bcd_decide 1/2 (||X||^2 - 2 <W, X H^T> + <W^T W, H H^T>) in fp64 (Gram identity, R25),
//                the l.17 branch and the extrapolation weights, on the device
//   k_bcd_commit V_m = V + w (V - V_prev), V_prev = V (accepted) or V_m = V_prev (correction)
//   k_bcd_commit_pq  P, Q = those of the new H (accepted) or of the rescaled H_prev
//   k_bcd_commit_h(_role)  the H side of the commit (float4 streams; the role variant swaps
//                the candidate / H_prev buffers instead of copying)
//   k_bcd_wside / k_bcd_post  one-CTA forms of the W side and of everything after the H pass
//                for small W (m r <= 8192, r <= 16)
// The X passes themselves are the MU kernels: k_fused / k_fused_c in their BCD mode (one pass
// per H half-iteration), their acc-only mode, or the fp16x2 tensor-core passes.
// Every decision stays on the device (state block `bs`, below), so one iteration is
// a fixed launch sequence the host captures once in a CUDA graph and replays.
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ntt {

namespace {

constexpr int BROWS = 128;

// test hook (ntt_debug_bcd_force_correct): the l.17 test of this iteration is treated as true
__device__ __forceinline__ bool forced_correction(const double* bs) {
  const uint64_t it = (uint64_t)bs[BS_IT];
  return it < 52 && (((uint64_t)bs[BS_FORCE] >> it) & 1ull);
}

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
#pragma unroll
      for (int l = 0; l < R; ++l) g += w[l] * Qs[l * R + k];  // Qs zero-padded beyond r
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
            double* __restrict__ Gpart, unsigned* __restrict__ maxw) {
  __shared__ float Wn[BROWS][R + 1];
  float mx = 0.0f;
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
    mx = fmaxf(mx, v);
    Wn[threadIdx.x][k] = v;
  }
  if (maxw) {  // max W for the fp16x2 scale of the W^T X pass (order-independent)
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxw, __float_as_uint(mx));
  }
  __syncthreads();
  const int rr = r * r;
  for (int t = threadIdx.x; t < rr; t += blockDim.x) {
    const int k = t / r, l = t % r;
    double s = 0.0;
    double s4[4] = {0.0, 0.0, 0.0, 0.0};  // four interleaved chains, fixed combination
#pragma unroll 4
    for (int q = 0; q < BROWS; ++q) s4[q & 3] += (double)Wn[q][k] * (double)Wn[q][l];
    s = (s4[0] + s4[1]) + (s4[2] + s4[3]);
    Gpart[(int64_t)blockIdx.x * rr + t] = s;
  }
}

// l.9 compensation on the H side without touching H: the logical H_m and H_prev are
// diag(sH[0..r)) Hm and diag(sH[R..R+r)) Hp (sH: [2][32]); their rows scale by c_k
__global__ void k_bcd_hscale(double* __restrict__ sH, int r, const double* __restrict__ c) {
  const int k = threadIdx.x;
  if (k < r && c[k] > 0.0) {
    sH[k] *= c[k];
    sH[32 + k] *= c[k];
    sH[64 + k] *= c[k];
  }
}

constexpr int BH_BN = 128;
constexpr int BH_MCH = 128;

// Spart[s][j][k] = sum_{i in rows of split s} W[i][k] X[i][j]; fp32 per 128-row chunk,
// fp64 across chunks.  Grid: (column tiles, splits).
template <int R>
__global__ void __launch_bounds__(BH_BN)
k_bcd_spart(const float* __restrict__ X, int64_t ldx, int64_t m, int64_t n, const float* __restrict__ W, int r,
            int64_t rows_per_split, double* __restrict__ Spart) {
  __shared__ float Ws[BH_MCH * R];
  const int64_t j = (int64_t)blockIdx.x * BH_BN + threadIdx.x;
  const bool valid = j < n;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_split;
  const int64_t r1 = min(m, r0 + rows_per_split);
  double Sd[R];
#pragma unroll
  for (int k = 0; k < R; ++k) Sd[k] = 0.0;
  for (int64_t c0 = r0; c0 < r1; c0 += BH_MCH) {
    const int rows = (int)min((int64_t)BH_MCH, r1 - c0);
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
    double* o = Spart + ((int64_t)blockIdx.y * n + j) * r;
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (k < r) o[k] = Sd[k];
  }
}

// S = W^T X and the H step in one pass when the rows are not split (short-wide X): thread j
// owns column j, S in fp32 per 128-row chunk and fp64 across (as k_bcd_spart), then
// H[:, j] = max(0, Hm - (G Hm - S) / L_H) with Hm = diag(sHm) Hm_stored, no S partials
template <int R>
__global__ void __launch_bounds__(BH_BN)
k_bcd_shup(const float* __restrict__ X, int64_t ldx, int64_t m, int64_t n, const float* __restrict__ W, int r,
           const double* __restrict__ G, const double* __restrict__ LH, const float* __restrict__ Hm,
           const double* __restrict__ sHm, float* __restrict__ H) {
  __shared__ float Ws[BH_MCH * R];
  __shared__ double Gs[R * R];
  for (int t = threadIdx.x; t < R * R; t += blockDim.x) {
    const int k = t / R, l = t % R;
    Gs[t] = (k < r && l < r) ? G[k * r + l] : 0.0;
  }
  const double L = *LH;
  const int64_t j = (int64_t)blockIdx.x * BH_BN + threadIdx.x;
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
  if (!valid) return;
  double hm[R];
#pragma unroll
  for (int k = 0; k < R; ++k) hm[k] = (k < r) ? (double)Hm[(int64_t)k * n + j] * sHm[k] : 0.0;
#pragma unroll
  for (int k = 0; k < R; ++k) {
    if (k < r) {
      double e = -Sd[k];
#pragma unroll
      for (int l = 0; l < R; ++l) e += Gs[k * R + l] * hm[l];
      const double v = L > 0.0 ? fmax(0.0, hm[k] - e / L) : hm[k];
      H[(int64_t)k * n + j] = (float)v;
    }
  }
}

// H = max(0, H_m - (G H_m - S) / L_H) per column j, S = sum_s Spart[s][j][:] (fixed order).
// The 128 columns of a block own a contiguous run of 128 r doubles in every split: each
// thread sums fixed elements of that run over the splits (coalesced), then reads its column
// back from shared memory.
template <int R>
__global__ void __launch_bounds__(BH_BN)
k_bcd_hup(const double* __restrict__ Spart, int nS, int64_t n, int r, const double* __restrict__ G,
          const double* __restrict__ LH, const float* __restrict__ Hm, const double* __restrict__ sHm,
          float* __restrict__ H, unsigned* __restrict__ maxh) {
  __shared__ double Gs[R * R];
  __shared__ double Ss[BH_BN * R];
  for (int t = threadIdx.x; t < R * R; t += blockDim.x) {
    const int k = t / R, l = t % R;
    Gs[t] = (k < r && l < r) ? G[k * r + l] : 0.0;
  }
  const double L = *LH;
  const int64_t nr = n * r;
  float mx = 0.0f;
  for (int64_t blk = blockIdx.x; blk * BH_BN < n; blk += gridDim.x) {
    const int64_t j0 = blk * BH_BN;
    const int cols = (int)min((int64_t)BH_BN, n - j0);
    const int len = cols * r;
    __syncthreads();  // the previous block's readers are done with Ss
    for (int e = threadIdx.x; e < len; e += BH_BN) Ss[e] = 0.0;
    for (int b = 0; b < nS; ++b) {  // split order, straight into shared memory (few registers)
      const double* src = Spart + (int64_t)b * nr + j0 * r;
      for (int e = threadIdx.x; e < len; e += BH_BN) Ss[e] += src[e];
    }
    __syncthreads();
    if (threadIdx.x < cols) {
      const int64_t j = j0 + threadIdx.x;
      double hm[R];
#pragma unroll
      for (int k = 0; k < R; ++k) hm[k] = (k < r) ? (double)Hm[(int64_t)k * n + j] * sHm[k] : 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (k < r) {
          double e = -Ss[threadIdx.x * r + k];
#pragma unroll
          for (int l = 0; l < R; ++l) e += Gs[k * R + l] * hm[l];
          const double v = L > 0.0 ? fmax(0.0, hm[k] - e / L) : hm[k];
          const float vf = (float)v;
          H[(int64_t)k * n + j] = vf;
          mx = fmaxf(mx, vf);
        }
      }
    }
  }
  if (maxh) {
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) atomicMax(maxh, __float_as_uint(mx));
  }
}

// P = sum_b Ppart[b] (fixed order) and the per-CTA partials of <W, P> (for the objective)
__global__ void __launch_bounds__(256)
k_bcd_psum_dot(const double* __restrict__ part, int nparts, int64_t len, const float* __restrict__ W,
               double* __restrict__ P, double* __restrict__ dotpart) {
  __shared__ double red[8];
  double d = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < len; t += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += part[(int64_t)b * len + t];
    P[t] = s;
    if (W) d += (double)W[t] * s;
  }
  if (!dotpart) return;
  d = warp_sum(d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = d;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    dotpart[blockIdx.x] = t;
  }
}

// lambda_max of a symmetric PSD r x r matrix M (r <= 32; the Lipschitz constants of R23).
// Repeated squaring A <- A^2 / max diag(A^2) drives A to the scaled projector onto the top
// eigenspace (stopped when A stops changing, at most 64 squarings = M^(2^64)); the Rayleigh
// quotient of M on the column of A with the largest diagonal entry is then lambda_max with an
// error quadratic in the eigenvector error.  Runs on the whole CTA (blockDim >= RP^2, a multiple
// of 32; thread (i, j) = (t / RP, t % RP) owns A[i][j]); the result is returned to every thread.
template <int RP>
struct SpecSmem {
  double A[RP][RP + 1];
  double Ms[RP][RP + 1];
  double red[32];
  double red2[32];
  double bc[2];
};

template <int RP>
__device__ double spec_dev(const double* __restrict__ M, int r, SpecSmem<RP>& S) {
  const int t = threadIdx.x, lane = t & 31, w = t >> 5, NWB = blockDim.x >> 5;
  const bool act = t < RP * RP;
  const int i = act ? t / RP : 0, j = act ? t % RP : 0;
  const bool in = act && i < r && j < r;
  const double mv = in ? M[i * r + j] : 0.0;
  __syncthreads();  // S may be reused from a previous call
  if (act) S.Ms[i][j] = mv;
  if (t < 32) S.red[t] = (t < r) ? M[t * r + t] : 0.0;
  __syncthreads();
  if (t < 32) {
    double d = S.red[t];
    for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
    if (t == 0) S.bc[0] = d;
  }
  __syncthreads();
  const double d0 = S.bc[0];
  if (!(d0 > 0.0)) return 0.0;  // PSD with a zero diagonal: M = 0 (uniform branch)
  if (act) S.A[i][j] = mv / d0;
  __syncthreads();
  for (int it = 0; it < 64; ++it) {
    double c = 0.0;
    if (act) {
#pragma unroll 8
      for (int k = 0; k < RP; ++k) c += S.A[i][k] * S.A[k][j];
    }
    __syncthreads();
    if (act && i == j) S.red[i] = c;
    __syncthreads();
    if (t < 32) {
      double d = (t < RP) ? S.red[t] : 0.0;
      for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
      if (t == 0) S.bc[0] = d;
    }
    __syncthreads();
    double diff = 0.0;
    if (act) {
      const double an = c / S.bc[0];
      diff = fabs(an - S.A[i][j]);
      S.A[i][j] = an;
    }
    for (int o = 16; o > 0; o >>= 1) diff = fmax(diff, __shfl_xor_sync(0xffffffffu, diff, o));
    if (lane == 0) S.red[w] = diff;
    __syncthreads();
    if (t < 32) {
      double d = (t < NWB) ? S.red[t] : 0.0;
      for (int o = 16; o > 0; o >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
      if (t == 0) S.bc[1] = d;
    }
    __syncthreads();
    // A entries are O(1) (max diagonal 1); a change <= 1e-12 means the non-top eigen-components
    // left are <= ~1e-12 (or within 1e-12 of lambda_max), and the Rayleigh quotient's error is
    // quadratic in them.  (A tighter stop would chase the ~1e-15 rounding noise of A^2.)
    if (S.bc[1] <= 1e-12) break;
  }
  // column with the largest diagonal entry (lowest index on ties)
  if (t < 32) {
    double d = (t < r) ? S.A[t][t] : -1.0;
    int idx = t;
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, d, o);
      const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
      if (od > d || (od == d && oi < idx)) {
        d = od;
        idx = oi;
      }
    }
    if (t == 0) S.bc[0] = (double)idx;
  }
  __syncthreads();
  const int jc = (int)S.bc[0];
  const double vi = act ? S.A[i][jc] : 0.0, vj = act ? S.A[j][jc] : 0.0;
  double num = in ? vi * S.Ms[i][j] * vj : 0.0;
  double den = (in && i == j) ? vi * vi : 0.0;
  num = warp_sum(num);
  den = warp_sum(den);
  __syncthreads();
  if (lane == 0) {
    S.red[w] = num;
    S.red2[w] = den;
  }
  __syncthreads();
  if (t == 0) {
    double sn = 0.0, sd = 0.0;
    for (int q = 0; q < NWB; ++q) {
      sn += S.red[q];
      sd += S.red2[q];
    }
    S.bc[0] = sd > 0.0 ? sn / sd : 0.0;
  }
  __syncthreads();
  return S.bc[0];
}

template <int RP>
__global__ void __launch_bounds__(RP * RP) k_spec_norm(const double* __restrict__ M, int r, double* __restrict__ out) {
  __shared__ SpecSmem<RP> S;
  const double v = spec_dev<RP>(M, r, S);
  if (threadIdx.x == 0) *out = v;
}

// ---- one-CTA stages for small W (m r <= 8192, r <= 16): the whole W side of an iteration
// and everything after the H pass except the H commit, so an iteration is 4-5 launches
constexpr int WS_T = 256;

// W side (l.5-10): L_W = ||Q||_2, W step, column L1 normalisation (W, W_prev; H_m, H_prev
// through their row scales), G = W^T W, L_H = ||G||_2.  Dynamic smem: m * RP floats.
template <int RP>
__global__ void __launch_bounds__(WS_T) k_bcd_wside(const float* __restrict__ Wm, float* __restrict__ W,
                                                    float* __restrict__ Wp, int m, int r, const double* __restrict__ Pc,
                                                    const double* __restrict__ Qc, double* __restrict__ bs,
                                                    double* __restrict__ c_out, double* __restrict__ G_out,
                                                    double* __restrict__ sH) {
  __shared__ SpecSmem<RP> S;
  __shared__ double Qs[RP * RP];
  __shared__ double cw[WS_T / 32][RP];
  __shared__ double cs[RP];
  __shared__ double Gp[WS_T];
  extern __shared__ float Wsm[];  // m x RP (the new W)
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  // the previous iteration's H commit stored H_m afresh (and H_prev when it accepted: copied, or
  // in the one-pass path by swapping the roles of the two H buffers -- done here, in thread 0)
  const bool prev_acc = bs[BS_ACC] != 0.0;
  if (t < 32) {
    if (bs[BS_FOLD] != 0.0) {
      // no H commit: the pass reads H_m = diag(a) B[1 - role] - diag(b) B[role] (after the swap
      // below).  Accepted: H_m = H + w_H (H - diag(s_p) H_prev) with H fresh in B[1 - role] and
      // the old H_prev in B[role]; correction: H_m = diag(s_p) H_prev.
      const double sp = sH[32 + t], wh = bs[BS_WH];
      sH[t] = prev_acc ? 1.0 + wh : sp;
      sH[64 + t] = prev_acc ? wh * sp : 0.0;
    } else {
      sH[t] = 1.0;
      sH[64 + t] = 0.0;
    }
    if (prev_acc) sH[32 + t] = 1.0;
  }
  __syncthreads();
  if (t == 0 && prev_acc) bs[BS_ROLE] = 1.0 - bs[BS_ROLE];
  const double LW = spec_dev<RP>(Qc, r, S);  // l.7
  if (t == 0) bs[BS_LW] = LW;
  for (int e = t; e < RP * RP; e += WS_T) {
    const int k = e / RP, l = e % RP;
    Qs[e] = (k < r && l < r) ? Qc[k * r + l] : 0.0;
  }
  __syncthreads();
  double csum[RP];
#pragma unroll
  for (int k = 0; k < RP; ++k) csum[k] = 0.0;
  for (int i = t; i < m; i += WS_T) {  // l.6-8, one row per thread
    double wv[RP];
#pragma unroll
    for (int k = 0; k < RP; ++k) wv[k] = (k < r) ? (double)Wm[i * r + k] : 0.0;
#pragma unroll
    for (int k = 0; k < RP; ++k) {
      float vf = 0.0f;
      if (k < r) {
        double g = -Pc[i * r + k];
#pragma unroll
        for (int l = 0; l < RP; ++l) g += wv[l] * Qs[l * RP + k];
        const double v = LW > 0.0 ? fmax(0.0, wv[k] - g / LW) : wv[k];
        vf = (float)v;
        csum[k] += (double)vf;
      }
      Wsm[i * RP + k] = vf;
    }
  }
#pragma unroll
  for (int k = 0; k < RP; ++k) {
    const double v = warp_sum(csum[k]);
    if (lane == 0) cw[w][k] = v;
  }
  __syncthreads();
  if (t < RP) {
    double sum = 0.0;
    for (int q = 0; q < WS_T / 32; ++q) sum += cw[q][t];
    cs[t] = sum;
    if (t < r) c_out[t] = sum;
  }
  __syncthreads();
  for (int e = t; e < m * r; e += WS_T) {  // l.9 (R24)
    const int i = e / r, k = e % r;
    const double ck = cs[k];
    float v = Wsm[i * RP + k];
    if (ck > 0.0) {
      v = (float)((double)v / ck);
      Wp[e] = (float)((double)Wp[e] / ck);
    }
    Wsm[i * RP + k] = v;
    W[e] = v;
  }
  if (t < r && cs[t] > 0.0) {
    sH[t] *= cs[t];
    sH[32 + t] *= cs[t];
    sH[64 + t] *= cs[t];
  }
  __syncthreads();
  constexpr int NE = RP * RP;
  constexpr int SPL = WS_T / NE >= 1 ? WS_T / NE : 1;  // row slices per G entry
  if (t < NE * SPL) {  // l.10: G = W^T W, fixed order
    const int e = t % NE, sl = t / NE, k = e / RP, l = e % RP;
    double g = 0.0;
    if (k < r && l < r)
      for (int i = sl; i < m; i += SPL) g += (double)Wsm[i * RP + k] * (double)Wsm[i * RP + l];
    Gp[t] = g;
  }
  __syncthreads();
  if (t < NE) {
    double g = 0.0;
    for (int sl = 0; sl < SPL; ++sl) g += Gp[sl * NE + t];
    const int k = t / RP, l = t % RP;
    if (k < r && l < r) G_out[k * r + l] = g;
  }
  __syncthreads();
  const double LH = spec_dev<RP>(G_out, r, S);
  if (t == 0) bs[BS_LH] = LH;
}

// After the H pass (l.15-27): P, Q of the candidate from their partials, the Gram-identity
// objective, the branch (as k_bcd_decide), and the W / P / Q commits.  Dynamic smem: m r doubles.
template <int RP>
__global__ void __launch_bounds__(WS_T) k_bcd_post(const double* __restrict__ Ppart, int nP,
                                                   const double* __restrict__ Qpart, int nQ, int m, int r,
                                                   const float* __restrict__ W, float* __restrict__ Wm,
                                                   float* __restrict__ Wp, double* __restrict__ Pc,
                                                   double* __restrict__ Qc, const double* __restrict__ c,
                                                   const double* __restrict__ G, double* __restrict__ bs,
                                                   double* __restrict__ trace) {
  extern __shared__ double Pn[];  // m r
  __shared__ double Qn[RP * RP];
  __shared__ double red[32], red2[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int mr = m * r, rr = r * r;
  double dot = 0.0, gq = 0.0;
  for (int e = t; e < mr; e += WS_T) {
    double sv = 0.0;
    for (int b = 0; b < nP; ++b) sv += Ppart[(int64_t)b * mr + e];
    Pn[e] = sv;
    dot += (double)W[e] * sv;
  }
  for (int e = t; e < rr; e += WS_T) {
    double sv = 0.0;
    for (int b = 0; b < nQ; ++b) sv += Qpart[(int64_t)b * rr + e];
    Qn[e] = sv;
    gq += G[e] * sv;
  }
  dot = warp_sum(dot);
  gq = warp_sum(gq);
  if (lane == 0) {
    red[w] = dot;
    red2[w] = gq;
  }
  __syncthreads();
  if (t == 0) {
    double s1 = 0.0, s2 = 0.0;
    for (int q = 0; q < WS_T / 32; ++q) {
      s1 += red[q];
      s2 += red2[q];
    }
    bs[BS_OBJNEW] = 0.5 * (bs[BS_XX] - 2.0 * s1 + s2);  // R25
    const double obj_new = bs[BS_OBJNEW], obj = bs[BS_OBJ], tt = bs[BS_T];
    if (obj_new < obj && !forced_correction(bs)) {  // l.21-27
      const double tp = (1.0 + sqrt(1.0 + 4.0 * tt * tt)) / 2.0;
      const double wgt = (tt - 1.0) / tp;
      const double LW = bs[BS_LW], LH = bs[BS_LH], dl = bs[BS_DELTA];
      bs[BS_WW] = fmin(wgt, dl * sqrt(bs[BS_LWP] / LW));
      bs[BS_WH] = fmin(wgt, dl * sqrt(bs[BS_LHP] / LH));
      bs[BS_ACC] = 1.0;
      bs[BS_LWP] = LW;
      bs[BS_LHP] = LH;
      bs[BS_T] = tp;
      bs[BS_OBJ] = obj_new;
    } else {  // l.17-20
      bs[BS_ACC] = 0.0;
      bs[BS_T] = 1.0;
    }
    const int it = (int)bs[BS_IT];
    if (trace) trace[it] = bs[BS_OBJ];
    bs[BS_IT] = (double)(it + 1);
  }
  __syncthreads();
  const bool acc = bs[BS_ACC] != 0.0;
  const double wW = bs[BS_WW];
  for (int e = t; e < mr; e += WS_T) {
    const int k = e % r;
    if (acc) {
      const double v = W[e], vp = Wp[e];
      Wm[e] = (float)(v + wW * (v - vp));
      Wp[e] = (float)v;
      Pc[e] = Pn[e];
    } else {
      Wm[e] = Wp[e];
      if (c[k] > 0.0) Pc[e] *= c[k];
    }
  }
  for (int e = t; e < rr; e += WS_T) {
    const int k = e / r, l = e % r;
    if (acc) Qc[e] = Qn[e];
    else Qc[e] *= (c[k] > 0.0 ? c[k] : 1.0) * (c[l] > 0.0 ? c[l] : 1.0);
  }
}

// l.17-27 on the device: accept (extrapolate) or correct; trace[it] = accepted objective
// (one warp) obj_new = 1/2 (||X||^2 - 2 <W, X H^T> + <W^T W, H H^T>) (Gram identity, R25) from
// the <W, P> partials of k_bcd_psum_dot; then the branch; clears the two fp16 max slots
__global__ void k_bcd_decide(double* __restrict__ bs, double* __restrict__ trace, const double* __restrict__ dotpart,
                             int ndot, const double* __restrict__ G, const double* __restrict__ Q, int rr,
                             unsigned* __restrict__ mxslots) {
  double s1 = 0.0, s2 = 0.0;
  for (int q = threadIdx.x; q < ndot; q += 32) s1 += dotpart[q];
  for (int q = threadIdx.x; q < rr; q += 32) s2 += G[q] * Q[q];
  s1 = warp_sum(s1);
  s2 = warp_sum(s2);
  if (threadIdx.x != 0) return;
  if (mxslots) {
    mxslots[0] = 0u;
    mxslots[1] = 0u;
  }
  bs[BS_OBJNEW] = 0.5 * (bs[BS_XX] - 2.0 * s1 + s2);
  const double obj_new = bs[BS_OBJNEW], obj = bs[BS_OBJ], t = bs[BS_T];
  if (obj_new < obj && !forced_correction(bs)) {
    const double tp = (1.0 + sqrt(1.0 + 4.0 * t * t)) / 2.0;
    const double w = (t - 1.0) / tp;
    const double LW = bs[BS_LW], LH = bs[BS_LH], dl = bs[BS_DELTA];
    bs[BS_WW] = fmin(w, dl * sqrt(bs[BS_LWP] / LW));  // fmin drops a NaN ratio (0/0) as min() does
    bs[BS_WH] = fmin(w, dl * sqrt(bs[BS_LHP] / LH));
    bs[BS_ACC] = 1.0;
    bs[BS_LWP] = LW;
    bs[BS_LHP] = LH;
    bs[BS_T] = tp;
    bs[BS_OBJ] = obj_new;
  } else {
    bs[BS_ACC] = 0.0;
    bs[BS_T] = 1.0;
  }
  const int it = (int)bs[BS_IT];
  if (trace) trace[it] = bs[BS_OBJ];
  bs[BS_IT] = (double)(it + 1);
}

// accepted: V_m = V + w (V - V_prev), V_prev = V;  correction: V_m = V_prev
__global__ void k_bcd_commit(const float* __restrict__ V, float* __restrict__ Vm, float* __restrict__ Vp, int64_t cnt,
                             const double* __restrict__ bs, int widx) {
  const bool acc = bs[BS_ACC] != 0.0;
  const double w = bs[widx];
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < cnt; e += (int64_t)gridDim.x * blockDim.x) {
    if (acc) {
      const double v = V[e], vp = Vp[e];
      Vm[e] = (float)(v + w * (v - vp));
      Vp[e] = (float)v;
    } else {
      Vm[e] = Vp[e];
    }
  }
}

// H side of l.18-27 with the scale vectors: Hp = diag(sHp) Hp_stored.  Accepted:
// Hm = H + w_H (H - Hp), Hp = H; correction: Hm = Hp.  Rows k over blockIdx.y; float4 columns
// when n % 4 == 0 (16-byte accesses: a streaming kernel needs the bytes in flight)
__global__ void k_bcd_commit_h(const float* __restrict__ H, float* __restrict__ Hm, float* __restrict__ Hp, int r,
                               int64_t n, const double* __restrict__ sH, const double* __restrict__ bs) {
  const bool acc = bs[BS_ACC] != 0.0;
  const double w = bs[BS_WH];
  const bool v4 = (n & 3) == 0;
  for (int k = blockIdx.y; k < r; k += gridDim.y) {
    const double sp = sH[32 + k];
    const int64_t base = (int64_t)k * n;
    if (v4) {
      const float4* H4 = reinterpret_cast<const float4*>(H + base);
      float4* Hm4 = reinterpret_cast<float4*>(Hm + base);
      float4* Hp4 = reinterpret_cast<float4*>(Hp + base);
      for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n / 4; j += (int64_t)gridDim.x * blockDim.x) {
        const float4 p4 = __ldcs(Hp4 + j);
        if (acc) {
          const float4 h4 = __ldcs(H4 + j);
          float4 m4;
          m4.x = (float)((double)h4.x + w * ((double)h4.x - (double)p4.x * sp));
          m4.y = (float)((double)h4.y + w * ((double)h4.y - (double)p4.y * sp));
          m4.z = (float)((double)h4.z + w * ((double)h4.z - (double)p4.z * sp));
          m4.w = (float)((double)h4.w + w * ((double)h4.w - (double)p4.w * sp));
          Hm4[j] = m4;
          Hp4[j] = h4;
        } else {
          Hm4[j] = make_float4((float)((double)p4.x * sp), (float)((double)p4.y * sp), (float)((double)p4.z * sp),
                               (float)((double)p4.w * sp));
        }
      }
    } else {
      for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double vp = (double)Hp[base + j] * sp;
        if (acc) {
          const double v = H[base + j];
          Hm[base + j] = (float)(v + w * (v - vp));
          Hp[base + j] = (float)v;
        } else {
          Hm[base + j] = (float)vp;
        }
      }
    }
  }
}

// Role-swapped variant of the H commit (one-pass path): the candidate lives in B[role], H_prev
// in B[1 - role].  Accepted: Hm = H + w_H (H - Hp) and the roles swap (k_bcd_wside flips
// BS_ROLE), so H_prev := H costs nothing; correction: Hm = Hp.  3 H-sized streams instead of 4.
__global__ void k_bcd_commit_h_role(const float* __restrict__ B0, const float* __restrict__ B1, float* __restrict__ Hm,
                                    int r, int64_t n, const double* __restrict__ sH, const double* __restrict__ bs) {
  const bool acc = bs[BS_ACC] != 0.0;
  const bool role = bs[BS_ROLE] != 0.0;
  const float* __restrict__ Hc = role ? B1 : B0;
  const float* __restrict__ Hp = role ? B0 : B1;
  const double w = bs[BS_WH];
  const bool v4 = (n & 3) == 0;
  for (int k = blockIdx.y; k < r; k += gridDim.y) {
    const double sp = sH[32 + k];
    const int64_t base = (int64_t)k * n;
    if (v4) {
      const float4* H4 = reinterpret_cast<const float4*>(Hc + base);
      const float4* P4 = reinterpret_cast<const float4*>(Hp + base);
      float4* M4 = reinterpret_cast<float4*>(Hm + base);
      for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n / 4; j += (int64_t)gridDim.x * blockDim.x) {
        const float4 p4 = __ldcs(P4 + j);
        float4 m4;
        if (acc) {
          const float4 h4 = __ldcs(H4 + j);
          m4.x = (float)((double)h4.x + w * ((double)h4.x - (double)p4.x * sp));
          m4.y = (float)((double)h4.y + w * ((double)h4.y - (double)p4.y * sp));
          m4.z = (float)((double)h4.z + w * ((double)h4.z - (double)p4.z * sp));
          m4.w = (float)((double)h4.w + w * ((double)h4.w - (double)p4.w * sp));
        } else {
          m4 = make_float4((float)((double)p4.x * sp), (float)((double)p4.y * sp), (float)((double)p4.z * sp),
                           (float)((double)p4.w * sp));
        }
        M4[j] = m4;
      }
    } else {
      for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        const double vp = (double)Hp[base + j] * sp;
        if (acc) {
          const double v = Hc[base + j];
          Hm[base + j] = (float)(v + w * (v - vp));
        } else {
          Hm[base + j] = (float)vp;
        }
      }
    }
  }
}

// final logical H_prev of the role-swapped path into B0 (the caller's H): after an accepted last
// iteration it is the candidate (pending swap, scale 1), otherwise B[1 - role] with its scale
__global__ void k_bcd_hout_role(float* __restrict__ B0, const float* __restrict__ B1, int r, int64_t n,
                                const double* __restrict__ sH, const double* __restrict__ bs) {
  const bool acc = bs[BS_ACC] != 0.0;
  const bool role = bs[BS_ROLE] != 0.0;
  const bool in_b1 = acc ? role : !role;
  const float* src = in_b1 ? B1 : B0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)r * n; e += (int64_t)gridDim.x * blockDim.x) {
    const float v = src[e];
    B0[e] = acc ? v : (float)((double)v * sH[32 + (int)(e / n)]);
  }
}

// out[k][j] = sH[32 + k] Hp[k][j] (the logical H_prev, returned at the end) or, with init,
// sH[0..64) = 1
__global__ void k_bcd_hout(const float* __restrict__ Hp, int r, int64_t n, double* __restrict__ sH,
                           float* __restrict__ out, int init, const double* __restrict__ bs) {
  if (init) {
    if (blockIdx.x == 0 && threadIdx.x < 96) sH[threadIdx.x] = threadIdx.x < 64 ? 1.0 : 0.0;
    return;
  }
  // after an accepted last iteration H_prev was stored afresh (its scale restarts at 1)
  const bool fresh = bs && bs[BS_ACC] != 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)r * n; e += (int64_t)gridDim.x * blockDim.x)
    out[e] = fresh ? Hp[e] : (float)((double)Hp[e] * sH[32 + (int)(e / n)]);
}

// accepted: P = X H^T, Q = H H^T of the new H (Pn, Qn).  Correction: H_prev was rescaled
// by c in l.9 (rows k x c_k), so X H_prev^T = P diag(c) and H_prev H_prev^T = diag(c) Q diag(c)
// (R26: the same matrices the oracle recomputes from H_prev, without another pass over X)
__global__ void k_bcd_commit_pq(double* __restrict__ Pc, const double* __restrict__ Pn, int64_t m, int r,
                                double* __restrict__ Qc, const double* __restrict__ Qn, const double* __restrict__ c,
                                const double* __restrict__ bs, double* __restrict__ sH) {
  const bool acc = bs[BS_ACC] != 0.0;
  if (blockIdx.x == 0 && threadIdx.x < 32) {  // Hm is stored fresh; Hp too when accepted
    sH[threadIdx.x] = 1.0;
    if (acc) sH[32 + threadIdx.x] = 1.0;
  }
  const int64_t mr = m * r, tot = mr + (int64_t)r * r;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    if (e < mr) {
      const int k = (int)(e % r);
      if (acc) Pc[e] = Pn[e];
      else if (c[k] > 0.0) Pc[e] *= c[k];
    } else {
      const int64_t q = e - mr;
      const int k = (int)(q / r), l = (int)(q % r);
      if (acc) Qc[q] = Qn[q];
      else Qc[q] *= (c[k] > 0.0 ? c[k] : 1.0) * (c[l] > 0.0 ? c[l] : 1.0);
    }
  }
}

__global__ void k_bcd_init(double* __restrict__ bs, double delta, double fold, double force) {
  if (threadIdx.x != 0) return;
  bs[BS_FORCE] = force;
  bs[BS_FOLD] = fold;
  bs[BS_OBJ] = 0.5 * bs[BS_XX];
  bs[BS_T] = 1.0;
  bs[BS_LWP] = bs[BS_LW];
  bs[BS_LHP] = bs[BS_LH];
  bs[BS_DELTA] = delta;
  bs[BS_IT] = 0.0;
  bs[BS_ACC] = 0.0;
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

// ||v||^2 of a rows x cols block (row stride ld), per-CTA fp64 partials.  Work items are
// (row, 4096-column chunk) pairs over the whole grid -- one CTA per row left all but `rows` SMs
// idle (16 ms for config 3's 32 x 2^25 X) -- with 128-bit streaming loads when aligned.
constexpr int SQ_CH = 4096;
__global__ void k_sumsq(const float* __restrict__ v, int64_t rows, int64_t cols, int64_t ld, double* __restrict__ part,
                        int evict_first) {
  double s = 0.0;
  const int64_t nch = (cols + SQ_CH - 1) / SQ_CH;
  const bool vec = ((reinterpret_cast<uintptr_t>(v) & 15) == 0) && ((ld & 3) == 0);
  for (int64_t c = blockIdx.x; c < rows * nch; c += gridDim.x) {
    const int64_t i = c / nch, j0 = (c - i * nch) * SQ_CH;
    const int64_t len = (cols - j0 < SQ_CH) ? cols - j0 : SQ_CH;
    const float* p = v + i * ld + j0;
    int64_t done = 0;
    if (vec) {
      const float4* p4 = reinterpret_cast<const float4*>(p);
      const int64_t n4 = len >> 2;
#pragma unroll 4
      for (int64_t q = threadIdx.x; q < n4; q += blockDim.x) {
        const float4 x = evict_first ? __ldcs(p4 + q) : __ldg(p4 + q);  // keep an L2-sized X for pq()
        s += (double)x.x * x.x + (double)x.y * x.y + (double)x.z * x.z + (double)x.w * x.w;
      }
      done = n4 << 2;
    }
    for (int64_t j = done + threadIdx.x; j < len; j += blockDim.x) {
      const double x = p[j];
      s += x * x;
    }
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

int rcls_bcd(int r) { return r <= 4 ? 4 : r <= 8 ? 8 : r <= 16 ? 16 : r <= 32 ? 32 : 64; }

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

cudaError_t launch_bcd_wnorm(float* W, float* Wp, int64_t m, int r, const double* c, double* Gpart, unsigned* maxw,
                             cudaStream_t st) {
  const unsigned g = (unsigned)bcd_w_ctas(m);
  switch (rcls_bcd(r)) {
    case 4: k_bcd_wnorm<4><<<g, BROWS, 0, st>>>(W, Wp, m, r, c, Gpart, maxw); break;
    case 8: k_bcd_wnorm<8><<<g, BROWS, 0, st>>>(W, Wp, m, r, c, Gpart, maxw); break;
    case 16: k_bcd_wnorm<16><<<g, BROWS, 0, st>>>(W, Wp, m, r, c, Gpart, maxw); break;
    default: k_bcd_wnorm<32><<<g, BROWS, 0, st>>>(W, Wp, m, r, c, Gpart, maxw); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_bcd_hscale(double* sH, int r, const double* c, cudaStream_t st) {
  k_bcd_hscale<<<1, 32, 0, st>>>(sH, r, c);
  return cudaGetLastError();
}

cudaError_t launch_bcd_commit_h(const float* H, float* Hm, float* Hp, int r, int64_t n, const double* sH,
                                const double* bs, cudaStream_t st) {
  const int64_t per = (n & 3) == 0 ? n / 4 : n;
  const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((per + 255) / 256, 2368 / std::max(r, 1) + 1));
  k_bcd_commit_h<<<dim3((unsigned)gx, (unsigned)r), 256, 0, st>>>(H, Hm, Hp, r, n, sH, bs);
  return cudaGetLastError();
}

cudaError_t launch_bcd_shup(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, int r, const double* G,
                            const double* LH, const float* Hm, const double* sHm, float* H, cudaStream_t st) {
  const unsigned g = (unsigned)((n + BH_BN - 1) / BH_BN);
  switch (rcls_bcd(r)) {
    case 4: k_bcd_shup<4><<<g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, G, LH, Hm, sHm, H); break;
    case 8: k_bcd_shup<8><<<g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, G, LH, Hm, sHm, H); break;
    case 16: k_bcd_shup<16><<<g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, G, LH, Hm, sHm, H); break;
    default: k_bcd_shup<32><<<g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, G, LH, Hm, sHm, H); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_bcd_hout(const float* Hp, int r, int64_t n, double* sH, float* out, int init, const double* bs,
                            cudaStream_t st) {
  k_bcd_hout<<<init ? 1 : 1184, 256, 0, st>>>(Hp, r, n, sH, out, init, bs);
  return cudaGetLastError();
}

bool bcd_cta_ok(int64_t m, int r) { return r <= 16 && m * (r <= 8 ? 8 : 16) <= 8192; }

cudaError_t launch_bcd_wside(const float* Wm, float* W, float* Wp, int m, int r, const double* Pc, const double* Qc,
                             double* bs, double* c, double* G, double* sH, cudaStream_t st) {
  if (r <= 8) {
    const size_t sm = sizeof(float) * (size_t)m * 8;
    k_bcd_wside<8><<<1, WS_T, sm, st>>>(Wm, W, Wp, m, r, Pc, Qc, bs, c, G, sH);
  } else {
    const size_t sm = sizeof(float) * (size_t)m * 16;
    k_bcd_wside<16><<<1, WS_T, sm, st>>>(Wm, W, Wp, m, r, Pc, Qc, bs, c, G, sH);
  }
  return cudaGetLastError();
}

cudaError_t launch_bcd_post(const double* Ppart, int nP, const double* Qpart, int nQ, int m, int r, const float* W,
                            float* Wm, float* Wp, double* Pc, double* Qc, const double* c, const double* G, double* bs,
                            double* trace, cudaStream_t st) {
  const size_t sm = sizeof(double) * (size_t)m * r;
  if (sm > 48 * 1024) {
    cudaError_t e = smem_optin((const void*)(r <= 8 ? k_bcd_post<8> : k_bcd_post<16>), sm);
    if (e) return e;
  }
  if (r <= 8) k_bcd_post<8><<<1, WS_T, sm, st>>>(Ppart, nP, Qpart, nQ, m, r, W, Wm, Wp, Pc, Qc, c, G, bs, trace);
  else k_bcd_post<16><<<1, WS_T, sm, st>>>(Ppart, nP, Qpart, nQ, m, r, W, Wm, Wp, Pc, Qc, c, G, bs, trace);
  return cudaGetLastError();
}

cudaError_t launch_bcd_commit_h_role(float* B0, float* B1, float* Hm, int r, int64_t n, const double* sH,
                                     const double* bs, cudaStream_t st) {
  const int64_t per = (n & 3) == 0 ? n / 4 : n;
  const int64_t gx = std::max<int64_t>(1, std::min<int64_t>((per + 255) / 256, 2368 / std::max(r, 1) + 1));
  k_bcd_commit_h_role<<<dim3((unsigned)gx, (unsigned)r), 256, 0, st>>>(B0, B1, Hm, r, n, sH, bs);
  return cudaGetLastError();
}

cudaError_t launch_bcd_hout_role(float* B0, float* B1, int r, int64_t n, const double* sH, const double* bs,
                                 cudaStream_t st) {
  k_bcd_hout_role<<<1184, 256, 0, st>>>(B0, B1, r, n, sH, bs);
  return cudaGetLastError();
}

int bcd_spart_splits(int64_t m, int64_t n, int num_sms) {
  const int64_t tiles = (n + BH_BN - 1) / BH_BN, chunks = (m + BH_MCH - 1) / BH_MCH;
  int64_t s = (4 * (int64_t)num_sms + tiles - 1) / tiles;  // >= 4 CTAs of 128 threads per SM
  s = std::max<int64_t>(1, std::min<int64_t>(s, chunks));
  return (int)std::min<int64_t>(s, 64);
}

cudaError_t launch_bcd_spart(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, int r, int nsplit,
                             double* Spart, cudaStream_t st) {
  const int64_t chunks = (m + BH_MCH - 1) / BH_MCH;
  const int64_t rps = ((chunks + nsplit - 1) / nsplit) * BH_MCH;
  const dim3 g((unsigned)((n + BH_BN - 1) / BH_BN), (unsigned)nsplit);
  switch (rcls_bcd(r)) {
    case 4: k_bcd_spart<4><<<g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, rps, Spart); break;
    case 8: k_bcd_spart<8><<<g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, rps, Spart); break;
    case 16: k_bcd_spart<16><<<g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, rps, Spart); break;
    case 32: k_bcd_spart<32><<<g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, rps, Spart); break;
    default: k_bcd_spart<64><<<g, BH_BN, 0, st>>>(X, ldx, m, n, W, r, rps, Spart); break;  // TT-SVD (r <= 64)
  }
  return cudaGetLastError();
}

cudaError_t launch_bcd_hup(const double* Spart, int nS, int64_t n, int r, const double* G, const double* LH,
                           const float* Hm, const double* sHm, float* H, unsigned* maxh, int num_sms, cudaStream_t st) {
  int64_t g = (n + BH_BN - 1) / BH_BN;
  if (g > 4 * num_sms) g = 4 * num_sms;
  switch (rcls_bcd(r)) {
    case 4: k_bcd_hup<4><<<(unsigned)g, BH_BN, 0, st>>>(Spart, nS, n, r, G, LH, Hm, sHm, H, maxh); break;
    case 8: k_bcd_hup<8><<<(unsigned)g, BH_BN, 0, st>>>(Spart, nS, n, r, G, LH, Hm, sHm, H, maxh); break;
    case 16: k_bcd_hup<16><<<(unsigned)g, BH_BN, 0, st>>>(Spart, nS, n, r, G, LH, Hm, sHm, H, maxh); break;
    default: k_bcd_hup<32><<<(unsigned)g, BH_BN, 0, st>>>(Spart, nS, n, r, G, LH, Hm, sHm, H, maxh); break;
  }
  return cudaGetLastError();
}

int bcd_dot_ctas(int64_t len, int num_sms) {
  const int64_t g = (len + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(g, 2 * (int64_t)num_sms));
}

cudaError_t launch_bcd_psum_dot(const double* part, int nparts, int64_t len, const float* W, double* P,
                                double* dotpart, int num_sms, cudaStream_t st) {
  k_bcd_psum_dot<<<(unsigned)bcd_dot_ctas(len, num_sms), 256, 0, st>>>(part, nparts, len, W, P, dotpart);
  return cudaGetLastError();
}

cudaError_t launch_spec_norm(const double* M, int r, double* out, cudaStream_t st) {
  if (r > 32) return cudaErrorInvalidValue;
  if (r <= 8) k_spec_norm<8><<<1, 64, 0, st>>>(M, r, out);
  else if (r <= 16) k_spec_norm<16><<<1, 256, 0, st>>>(M, r, out);
  else k_spec_norm<32><<<1, 1024, 0, st>>>(M, r, out);
  return cudaGetLastError();
}

cudaError_t launch_bcd_init(double* bs, double delta, bool fold, uint64_t force, cudaStream_t st) {
  k_bcd_init<<<1, 32, 0, st>>>(bs, delta, fold ? 1.0 : 0.0, (double)force);
  return cudaGetLastError();
}

cudaError_t launch_bcd_decide(double* bs, double* trace, const double* dotpart, int ndot, const double* G,
                              const double* Q, int r, unsigned* mxslots, cudaStream_t st) {
  k_bcd_decide<<<1, 32, 0, st>>>(bs, trace, dotpart, ndot, G, Q, r * r, mxslots);
  return cudaGetLastError();
}

cudaError_t launch_bcd_commit(const float* V, float* Vm, float* Vp, int64_t cnt, const double* bs, int widx,
                              cudaStream_t st) {
  const int64_t g = std::min<int64_t>(1184, (cnt + 255) / 256);
  k_bcd_commit<<<(unsigned)std::max<int64_t>(g, 1), 256, 0, st>>>(V, Vm, Vp, cnt, bs, widx);
  return cudaGetLastError();
}

cudaError_t launch_bcd_commit_pq(double* Pc, const double* Pn, int64_t m, int r, double* Qc, const double* Qn,
                                 const double* c, const double* bs, double* sH, cudaStream_t st) {
  const int64_t tot = m * r + (int64_t)r * r;
  const int64_t g = std::min<int64_t>(1184, (tot + 255) / 256);
  k_bcd_commit_pq<<<(unsigned)g, 256, 0, st>>>(Pc, Pn, m, r, Qc, Qn, c, bs, sH);
  return cudaGetLastError();
}

cudaError_t launch_scale_copy(const float* src, float* a, float* b, int64_t cnt, const double* num, const double* den,
                              cudaStream_t st) {
  k_scale_copy<<<1184, 256, 0, st>>>(src, a, b, cnt, num, den);
  return cudaGetLastError();
}

int sumsq_ctas() { return 1184; }

cudaError_t launch_sumsq(const float* v, int64_t rows, int64_t cols, int64_t ld, double* part, cudaStream_t st,
                         bool evict_first) {
  k_sumsq<<<1184, 256, 0, st>>>(v, rows, cols, ld, part, evict_first ? 1 : 0);
  return cudaGetLastError();
}

}  // namespace ntt
