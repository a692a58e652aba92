// tt_rank.cu -- the SVD rank rule of Alg. 2 l.5-6 (section III-A P:194;
// SURVEY s.8(f) f2) on the GPU:
//   r_l = smallest k in [1, N] with sqrt(s_{k+1}^2 + ... + s_N^2) / sqrt(sum s_i^2) <= eps
// for the current unfolding X (m x n, N = min(m, n)).  The squared singular values
// are the eigenvalues of the Gram matrix C = X X^T (m <= 512; padded with m - n
// zeros when n < m) or C = X^T X (n <= 512 < m):
//   k_gram         split-K tiles of C, fp64 FMA on the fp32 inputs (exact products), fixed order
//   k_gram_sum     fixed-order sum of the split partials, symmetric fill
//   k_eig_rank     ONE CTA: Householder tridiagonalisation of C (fp64, matrix in global /
//                  L2), Sturm-count bisection for every eigenvalue, then the tail rule
// Gram-based eigenvalues carry an absolute error ~1e-16 * trace(C), so the rule is
// exact for eps >= ~1e-7 (reading R21).  Deterministic (fixed reduction orders).
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ntt {

namespace {

constexpr int kRankOneCta = 512;  // the one-CTA eigensolver up to this size, the grid path above
constexpr int GT = 32;   // Gram output tile (GT x GT)
constexpr int GK = 32;   // columns of the long dimension per smem block

// C tile (ta, tb) (tb >= ta) over the split's range of the long index t:
// u_t[a] = X[a * sa + t * st]  (X X^T: sa = ldx, st = 1;  X^T X: sa = 1, st = ldx)
// 64 threads, 4 x 4 outputs each (rows ty + 8u, columns tx + 8v): 8 shared loads per 16
// fp64 FMAs, so the FP64 pipe, not shared memory, sets the rate.
constexpr int GTH = 64;
__global__ void __launch_bounds__(GTH)
k_gram(const float* __restrict__ X, int64_t sa, int64_t st, int N, int64_t T, int ntile, int64_t chunk,
       double* __restrict__ part) {
  // fp64 in shared memory: each element is converted once when staged, not per use
  __shared__ double As[GK][GT + 1];
  __shared__ double Bs[GK][GT + 1];
  // upper-triangular tile index -> (ta, tb)
  int tix = blockIdx.x, ta = 0;
  while (tix >= ntile - ta) {
    tix -= ntile - ta;
    ++ta;
  }
  const int tb = ta + tix;
  const int split = blockIdx.y;
  const int64_t t0 = (int64_t)split * chunk, t1 = min(T, t0 + chunk);
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  double acc[4][4];
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
  for (int64_t tb0 = t0; tb0 < t1; tb0 += GK) {
    for (int e = threadIdx.x; e < GT * GK; e += GTH) {
      // XX^T: consecutive threads along t (contiguous); X^T X: along a (contiguous)
      int i, k;
      if (st == 1) {
        i = e / GK;
        k = e % GK;
      } else {
        i = e % GT;
        k = e / GT;
      }
      const int64_t t = tb0 + k;
      const int a = ta * GT + i, bb = tb * GT + i;
      As[k][i] = (t < t1 && a < N) ? (double)X[(int64_t)a * sa + t * st] : 0.0;
      Bs[k][i] = (t < t1 && bb < N) ? (double)X[(int64_t)bb * sa + t * st] : 0.0;
    }
    __syncthreads();
    // fp64 FMA: the product of two fp32 values is exact in fp64, so the Gram (and the
    // eigenvalues) carry ~1e-16 relative error instead of fp32's ~1e-7
#pragma unroll 4
    for (int k = 0; k < GK; ++k) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = As[k][ty + 8 * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) b[v] = Bs[k][tx + 8 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
  // part[split][tile][GT][GT]
  const int tile = blockIdx.x;
  double* dst = part + ((int64_t)split * gridDim.x + tile) * (GT * GT);
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) dst[(ty + 8 * u) * GT + tx + 8 * v] = acc[u][v];
}

// one warp per entry of the upper tiles: lanes take every 32nd split, fixed shuffle tree
__global__ void k_gram_sum(const double* __restrict__ part, int nsplit, int ntile, int N, double* __restrict__ C) {
  const int nut = ntile * (ntile + 1) / 2;
  const int64_t nent = (int64_t)nut * GT * GT;
  const int lane = threadIdx.x & 31;
  for (int64_t e = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; e < nent;
       e += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    int tix = (int)(e / (GT * GT));
    const int w = (int)(e % (GT * GT));
    const int tile = tix;
    int ta = 0;
    while (tix >= ntile - ta) {
      tix -= ntile - ta;
      ++ta;
    }
    const int tb = ta + tix;
    const int a = ta * GT + w / GT, b = tb * GT + w % GT;
    if (a >= N || b >= N) continue;  // warp-uniform
    double s = 0.0;
    for (int sp = lane; sp < nsplit; sp += 32) s += part[((int64_t)sp * nut + tile) * (GT * GT) + w];
    s = warp_sum(s);
    if (lane == 0) {
      C[(int64_t)a * N + b] = s;
      C[(int64_t)b * N + a] = s;
    }
  }
}

// ---------------------------------------------------------------- eigen + rule
constexpr int ET = 1024;

__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (threadIdx.x < (int)(blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    s = warp_sum(s);
    if (threadIdx.x == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

// number of eigenvalues of the symmetric tridiagonal (d, e) strictly below x
__device__ int sturm_count(const double* d, const double* e2, int N, double x) {
  int c = 0;
  double q = d[0] - x;
  if (q < 0.0) ++c;
  for (int i = 1; i < N; ++i) {
    if (q == 0.0) q = 1e-300;
    q = (d[i] - x) - e2[i - 1] / q;
    if (q < 0.0) ++c;
  }
  return c;
}

// One CTA.  C: N x N symmetric (destroyed).  v, p: N doubles scratch (global).
// out: eig[N] ascending (optional), rank[0] = r for tt_eps.
__global__ void __launch_bounds__(ET)
k_eig_rank(double* __restrict__ C, int N, double* __restrict__ vg, double* __restrict__ pg, double tt_eps,
           double* __restrict__ eig, int* __restrict__ rank_out) {
  extern __shared__ double sm[];
  double* d = sm;           // N
  double* e = d + N;        // N
  double* e2 = e + N;       // N
  double* lam = e2 + N;     // N
  vg = lam + N;             // N: Householder vector and p, in shared memory
  pg = vg + N;              // N (the global vg / pg arguments are not used)
  double* red = pg + N;     // 33
  const int tid = threadIdx.x, T = blockDim.x;
  // ---- Householder tridiagonalisation, H = I - 2 v v^T with ||v|| = 1
  for (int k = 0; k + 2 < N; ++k) {
    const int L = N - k - 1;        // trailing size
    double* A = C + (int64_t)(k + 1) * N + (k + 1);  // A'[i][j] = A[i * N + j]
    // x = C[k+1 .. N-1][k]
    double xs = 0.0;
    for (int i = tid; i < L; i += T) {
      const double xi = C[(int64_t)(k + 1 + i) * N + k];
      vg[i] = xi;
      xs += xi * xi;
    }
    const double nx2 = block_sum(xs, red);
    const double x0 = vg[0];
    const double nx = sqrt(nx2);
    const double alpha = (x0 > 0.0) ? -nx : nx;
    // v = x - alpha e1, ||v||^2 = nx2 - 2 alpha x0 + alpha^2
    const double nv2 = nx2 - 2.0 * alpha * x0 + alpha * alpha;
    if (tid == 0) {
      d[k] = C[(int64_t)k * N + k];
      e[k] = (nx2 > 0.0) ? alpha : 0.0;
    }
    if (nv2 <= 0.0 || nx2 == 0.0) {  // already reduced
      __syncthreads();
      if (tid == 0) e[k] = vg[0];
      __syncthreads();
      continue;
    }
    const double inv = 1.0 / sqrt(nv2);
    __syncthreads();
    for (int i = tid; i < L; i += T) vg[i] = (i == 0 ? vg[0] - alpha : vg[i]) * inv;
    __syncthreads();
    // p = A' v (warp per row, lanes over columns)
    const int w = tid >> 5, ln = tid & 31, nw = T >> 5;
    for (int i = w; i < L; i += nw) {
      double s = 0.0;
      for (int j = ln; j < L; j += 32) s += A[(int64_t)i * N + j] * vg[j];
      s = warp_sum(s);
      if (ln == 0) pg[i] = s;
    }
    __syncthreads();
    double kp = 0.0;
    for (int i = tid; i < L; i += T) kp += vg[i] * pg[i];
    const double K = block_sum(kp, red);
    for (int i = tid; i < L; i += T) pg[i] = pg[i] - K * vg[i];  // w = p - K v
    __syncthreads();
    // A' -= 2 (v w^T + w v^T)
    for (int q = tid; q < L * L; q += T) {  // L <= 511: 32-bit index math
      const int i = q / L, j = q - i * L;
      A[(int64_t)i * N + j] -= 2.0 * (vg[i] * pg[j] + pg[i] * vg[j]);
    }
    __syncthreads();
  }
  if (tid == 0) {
    if (N >= 2) {
      d[N - 2] = C[(int64_t)(N - 2) * N + (N - 2)];
      e[N - 2] = C[(int64_t)(N - 1) * N + (N - 2)];
    }
    d[N - 1] = C[(int64_t)(N - 1) * N + (N - 1)];
  }
  __syncthreads();
  for (int i = tid; i < N - 1; i += T) e2[i] = e[i] * e[i];
  __syncthreads();
  // ---- Gershgorin bounds, then bisection for eigenvalue index i (ascending)
  double gl = 1e300, gu = -1e300;
  if (tid == 0) {
    for (int i = 0; i < N; ++i) {
      const double rad = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < N ? fabs(e[i]) : 0.0);
      gl = fmin(gl, d[i] - rad);
      gu = fmax(gu, d[i] + rad);
    }
    red[0] = gl;
    red[1] = gu;
  }
  __syncthreads();
  gl = red[0];
  gu = red[1];
  const double span = fmax(gu - gl, 1e-300);
  for (int i = tid; i < N; i += T) {
    double lo = gl - 1e-12 * span, hi = gu + 1e-12 * span;
    for (int it = 0; it < 200 && hi - lo > 1e-15 * fmax(fabs(lo), fabs(hi)) + 1e-300; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (sturm_count(d, e2, N, mid) <= i) lo = mid;
      else hi = mid;
    }
    lam[i] = fmax(0.5 * (lo + hi), 0.0);  // PSD: clamp round-off negatives
  }
  __syncthreads();
  if (tid == 0) {
    // tail after k (descending order) = sum of the N - k smallest, accumulated from the smallest
    double tot = 0.0;
    for (int i = 0; i < N; ++i) tot += lam[i];
    int r = N;
    if (tot <= 0.0) {
      r = 1;
    } else {
      double asc = 0.0;  // sum of the j smallest
      // k = N - j: condition sqrt(asc_j / tot) <= eps; smallest k <=> largest j
      int best = 0;
      for (int j = 1; j < N; ++j) {
        asc += lam[j - 1];
        if (sqrt(asc / tot) <= tt_eps) best = j;
        else break;
      }
      r = N - best;
    }
    rank_out[0] = r;
  }
  if (eig)
    for (int i = tid; i < N; i += T) eig[i] = lam[i];
}

// ------------------------------------------- N > 512: the same algorithm on the whole grid
// (SURVEY s.8(f) f2 at the paper's 256^4 scale, whose step 2 has min(m, n) = 2560).  The matrix
// (fp64, up to 4096^2 = 128 MB) stays in global memory / L2; every step of the Householder
// reduction is split across all CTAs of one cooperative launch:
//   every CTA   x = row k of the trailing matrix (= column k by symmetry, contiguous), ||x||, v
//               (redundantly: no barrier needed for v)
//   warp-rows   p_i = sum_j A'[i][j] v_j for the rows this warp owns (row i -> global warp i % W)
//   -- grid barrier --
//   every CTA   K = v^T p, w = p - K v (redundantly)
//   warp-rows   A'[i][j] -= 2 (v_i w_j + w_i v_j)
//   -- grid barrier --
// with the arithmetic of k_eig_rank (same reflector, same update formula; the row sums are
// lane-strided warp sums instead of one warp per row of a 1024-thread CTA, so the tridiagonal
// agrees to rounding).  Eigenvalues: k_bisect_grid, a warp per eigenvalue, 32-point
// multisection with the Sturm count of k_eig_rank.
constexpr int TG_T = 256;

__device__ __forceinline__ void tg_barrier(unsigned* ctr, unsigned& epoch) {
  __syncthreads();
  epoch += gridDim.x;
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < epoch);
    __threadfence();
  }
  __syncthreads();
}

__global__ void __launch_bounds__(TG_T)
k_tridiag_grid(double* __restrict__ C, int N, double* __restrict__ pg, double* __restrict__ dg,
               double* __restrict__ eg, unsigned* __restrict__ ctr, double* __restrict__ Vh) {
  extern __shared__ double tsm[];
  double* v = tsm;      // N
  double* w = v + N;    // N
  __shared__ double red[33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = gridDim.x * (TG_T / 32);
  const int gw = blockIdx.x * (TG_T / 32) + warp;
  unsigned epoch = 0;
  for (int k = 0; k + 2 < N; ++k) {
    const int L = N - k - 1;
    const double* xrow = C + (int64_t)k * N + (k + 1);
    double xs = 0.0;
    for (int j = tid; j < L; j += TG_T) {
      const double xj = __ldcg(xrow + j);
      v[j] = xj;
      xs += xj * xj;
    }
    const double nx2 = block_sum(xs, red);
    const double x0 = v[0];
    const double nx = sqrt(nx2);
    const double alpha = (x0 > 0.0) ? -nx : nx;
    const double nv2 = nx2 - 2.0 * alpha * x0 + alpha * alpha;
    if (blockIdx.x == 0 && tid == 0) {
      dg[k] = __ldcg(C + (int64_t)k * N + k);
      eg[k] = (nx2 > 0.0) ? alpha : 0.0;
    }
    if (nv2 <= 0.0 || nx2 == 0.0) {  // already reduced (every CTA takes this branch)
      if (blockIdx.x == 0 && tid == 0) eg[k] = x0;
      if (Vh && blockIdx.x == 0)  // identity reflector (TT-SVD back-transformation)
        for (int j = tid; j < L; j += TG_T) Vh[(int64_t)k * N + j] = 0.0;
      __syncthreads();
      continue;
    }
    const double inv = 1.0 / sqrt(nv2);
    __syncthreads();
    for (int j = tid; j < L; j += TG_T) v[j] = (j == 0 ? v[0] - alpha : v[j]) * inv;
    __syncthreads();
    if (Vh && blockIdx.x == 0)  // the reflector, kept for the TT-SVD back-transformation (row k)
      for (int j = tid; j < L; j += TG_T) Vh[(int64_t)k * N + j] = v[j];
    for (int i = gw; i < L; i += W) {
      const double* row = C + (int64_t)(k + 1 + i) * N + (k + 1);
      double a0 = 0.0, a1 = 0.0;
      int j = lane;
      for (; j + 32 < L; j += 64) {
        a0 = fma(__ldcg(row + j), v[j], a0);
        a1 = fma(__ldcg(row + j + 32), v[j + 32], a1);
      }
      if (j < L) a0 = fma(__ldcg(row + j), v[j], a0);
      const double sum = warp_sum(a0 + a1);
      if (lane == 0) pg[i] = sum;
    }
    tg_barrier(ctr, epoch);
    double kp = 0.0;
    for (int j = tid; j < L; j += TG_T) {
      const double pj = __ldcg(pg + j);
      w[j] = pj;
      kp += v[j] * pj;
    }
    const double K = block_sum(kp, red);
    for (int j = tid; j < L; j += TG_T) w[j] = w[j] - K * v[j];
    __syncthreads();
    for (int i = gw; i < L; i += W) {
      double* row = C + (int64_t)(k + 1 + i) * N + (k + 1);
      const double vi = v[i], wi = w[i];
      for (int j = lane; j < L; j += 32) row[j] = __ldcg(row + j) - 2.0 * (vi * w[j] + wi * v[j]);
    }
    tg_barrier(ctr, epoch);
  }
  if (blockIdx.x == 0 && tid == 0) {
    if (N >= 2) {
      dg[N - 2] = __ldcg(C + (int64_t)(N - 2) * N + (N - 2));
      eg[N - 2] = __ldcg(C + (int64_t)(N - 1) * N + (N - 2));
    }
    dg[N - 1] = __ldcg(C + (int64_t)(N - 1) * N + (N - 1));
  }
}

// number of eigenvalues of the tridiagonal (d, e) strictly below x (k_eig_rank's sturm_count
// with e^2 formed on the fly)
__device__ int sturm_count_e(const double* __restrict__ d, const double* __restrict__ e, int N, double x) {
  int c = 0;
  double q = d[0] - x;
  if (q < 0.0) ++c;
  for (int i = 1; i < N; ++i) {
    if (q == 0.0) q = 1e-300;
    q = (d[i] - x) - (e[i - 1] * e[i - 1]) / q;
    if (q < 0.0) ++c;
  }
  return c;
}

// lam[i] (ascending) for every i: a warp per eigenvalue, each round evaluates the Sturm count at
// 32 interior points of [lo, hi] (one per lane) and keeps the 1/33 sub-interval that holds
// eigenvalue i; stops at the bisection tolerance of k_eig_rank.
__global__ void __launch_bounds__(256) k_bisect_grid(const double* __restrict__ d, const double* __restrict__ e, int N,
                                                    double* __restrict__ lam) {
  const int lane = threadIdx.x & 31;
  const int gwarp = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)(((int64_t)gridDim.x * blockDim.x) >> 5);
  double gl = 1e300, gu = -1e300;
  for (int i = lane; i < N; i += 32) {
    const double rad = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < N ? fabs(e[i]) : 0.0);
    gl = fmin(gl, d[i] - rad);
    gu = fmax(gu, d[i] + rad);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gl = fmin(gl, __shfl_xor_sync(0xffffffffu, gl, o));
    gu = fmax(gu, __shfl_xor_sync(0xffffffffu, gu, o));
  }
  const double span = fmax(gu - gl, 1e-300);
  for (int idx = gwarp; idx < N; idx += nwarps) {
    double lo = gl - 1e-12 * span, hi = gu + 1e-12 * span;
    for (int it = 0; it < 64 && hi - lo > 1e-15 * fmax(fabs(lo), fabs(hi)) + 1e-300; ++it) {
      const double wdt = hi - lo;
      const double x = lo + wdt * (double)(lane + 1) / 33.0;
      const unsigned above = __ballot_sync(0xffffffffu, sturm_count_e(d, e, N, x) > idx);
      const int l = above ? __ffs(above) - 1 : 32;
      const double nlo = lo + wdt * (double)l / 33.0;
      const double nhi = (l == 32) ? hi : lo + wdt * (double)(l + 1) / 33.0;
      lo = nlo;
      hi = nhi;
    }
    if (lane == 0) lam[idx] = fmax(0.5 * (lo + hi), 0.0);  // PSD: clamp round-off negatives
  }
}

// the tail rule of k_eig_rank on ascending eigenvalues (one thread)
__global__ void k_rank_from_eig(const double* __restrict__ lam, int N, double tt_eps, int* __restrict__ rank_out,
                                double* __restrict__ eig) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double tot = 0.0;
    for (int i = 0; i < N; ++i) tot += lam[i];
    int r = N;
    if (tot <= 0.0) {
      r = 1;
    } else {
      double asc = 0.0;
      int best = 0;
      for (int j = 1; j < N; ++j) {
        asc += lam[j - 1];
        if (sqrt(asc / tot) <= tt_eps) best = j;
        else break;
      }
      r = N - best;
    }
    rank_out[0] = r;
  }
  if (eig)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) eig[i] = lam[i];
}

}  // namespace

size_t rank_rule_bytes(int64_t N, int64_t T, int num_sms) {
  const int ntile = (int)((N + GT - 1) / GT);
  const int nut = ntile * (ntile + 1) / 2;
  int64_t nsplit = (8 * num_sms + nut - 1) / nut;
  int64_t ch = (T + nsplit - 1) / nsplit;
  ch = (ch + GK - 1) / GK * GK;
  nsplit = (T + ch - 1) / ch;
  return sizeof(double) * ((size_t)nsplit * nut * GT * GT + (size_t)N * N + 4 * (size_t)N + 64) + 64;
}

cudaError_t launch_gram(const float* X, int64_t m, int64_t n, int64_t ldx, char* ws, int num_sms, double** Cout,
                        cudaStream_t st) {
  const bool rows = m <= n;  // C = X X^T (N = m) or X^T X (N = n)
  const int N = (int)(rows ? m : n);
  const int64_t T = rows ? n : m;
  const int64_t sa = rows ? ldx : 1, stt = rows ? 1 : ldx;
  const int ntile = (N + GT - 1) / GT;
  const int nut = ntile * (ntile + 1) / 2;
  int64_t nsplit = (8 * num_sms + nut - 1) / nut;
  int64_t chunk = (T + nsplit - 1) / nsplit;
  chunk = (chunk + GK - 1) / GK * GK;
  nsplit = (T + chunk - 1) / chunk;
  double* part = reinterpret_cast<double*>(ws);
  double* C = part + (size_t)nsplit * nut * GT * GT;
  *Cout = C;
  k_gram<<<dim3((unsigned)nut, (unsigned)nsplit), GTH, 0, st>>>(X, sa, stt, N, T, ntile, chunk, part);
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  k_gram_sum<<<1184, 256, 0, st>>>(part, (int)nsplit, ntile, N, C);
  return cudaGetLastError();
}

cudaError_t launch_rank_rule(const float* X, int64_t m, int64_t n, int64_t ldx, double tt_eps, char* ws,
                             int num_sms, int* d_rank, double* d_eig, cudaStream_t st) {
  const int N = (int)(m <= n ? m : n);
  double* C = nullptr;
  cudaError_t e = launch_gram(X, m, n, ldx, ws, num_sms, &C, st);
  if (e) return e;
  double* vg = C + (size_t)N * N;
  double* pg = vg + N;
  if (N <= kRankOneCta) {
    const size_t sm = sizeof(double) * (6 * (size_t)N + 40);
    e = smem_optin((const void*)(k_eig_rank), sm);
    if (e) return e;
    k_eig_rank<<<1, ET, sm, st>>>(C, N, vg, pg, tt_eps, d_eig, d_rank);
    return cudaGetLastError();
  }
  // grid path: p (N, at vg) | d (N) | e (N) | lam (N) | barrier counter, after C (4 N + 64 doubles)
  double* dg = vg + N;
  double* eg = dg + N;
  double* lam = eg + N;
  unsigned* ctr = reinterpret_cast<unsigned*>(lam + N);
  e = launch_tridiag_eig(C, N, vg, dg, eg, lam, ctr, nullptr, num_sms, st);
  if (e) return e;
  k_rank_from_eig<<<1, 256, 0, st>>>(lam, N, tt_eps, d_rank, d_eig);
  return cudaGetLastError();
}

cudaError_t launch_tridiag_eig(double* C, int N, double* p, double* d, double* e, double* lam, unsigned* ctr,
                               double* Vh, int num_sms, cudaStream_t st) {
  cudaError_t err = cudaMemsetAsync(ctr, 0, 64, st);
  if (err) return err;
  const size_t sm = sizeof(double) * 2 * (size_t)N;
  err = smem_optin((const void*)(k_tridiag_grid), sm);
  if (err) return err;
  int per_sm = 0;
  err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tridiag_grid, TG_T, sm);
  if (err) return err;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  const int grid = num_sms * std::min(per_sm, 2);
  int Ni = N;
  void* args[] = {&C, &Ni, &p, &d, &e, &ctr, &Vh};
  err = cudaLaunchCooperativeKernel((const void*)k_tridiag_grid, dim3(grid), dim3(TG_T), args, sm, st);
  if (err) return err;
  k_bisect_grid<<<(unsigned)std::min<int64_t>((N + 7) / 8, 4 * num_sms), 256, 0, st>>>(d, e, N, lam);
  return cudaGetLastError();
}

}  // namespace ntt
