// tt_svd.cu -- the TT-SVD baseline (unconstrained TT by sequential truncated SVDs; the
// comparison method of P:78; SURVEY s.8(f) f4; reading R28) on the GPU.
// Per TT step the current matrix X (m x n, N = min(m, n) <= 512) goes through
//   Gram           C = X X^T (m <= n) or X^T X (m > n), fp64 (tt_rank.cu: k_gram)
//   k_svd_eig      ONE CTA: Householder tridiagonalisation T = Q^T C Q (reflectors kept),
//                  Sturm bisection for every eigenvalue, the tail rule (Alg. 2 l.5-6) for
//                  r, inverse iteration on T for the top r eigenvalues (one thread per
//                  vector, LU with partial pivoting), CGS2 orthonormalisation, a
//                  Rayleigh-Ritz step (parallel Jacobi on Y^T T Y, r x r, in shared
//                  memory) and the back-transformation u = Q y
//   m <= n:        core = U_r (sign convention: the largest |entry| of a column > 0),
//                  X' = U_r^T X (split-K k_bcd_spart + k_rows_from_spart)
//   m > n:         core = X V_r diag(1/s) (k_xht_partial), X' = diag(s) V_r^T, same signs
// The next step's matrix is X' reshaped (row-major, no data movement).
#include <algorithm>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ntt {

namespace {

constexpr int ST = 1024;
constexpr int RMAX = 64;

__device__ double blk_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double s = (threadIdx.x < (int)(blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    s = warp_sum(s);
    if (threadIdx.x == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

__device__ int sturm(const double* d, const double* e2, int N, double x) {
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

__device__ __forceinline__ double start_value(int i, int k) {
  uint64_t z = (uint64_t)i * 0x9E3779B97F4A7C15ull + (uint64_t)(k + 1) * 0xD1B54A32D192ED03ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;  // [-1, 1)
}

// Steps 3-9 of the TT-SVD eigensolver on the tridiagonal T = (d, e) with its ascending eigenvalues
// lam[N] (all in shared memory): the tail rule and cap -> r; inverse iteration for the top r
// eigenvalues; CGS2; Rayleigh-Ritz (parallel Jacobi on Y^T T Y); Ritz order; Z = Y Q sorted
// (vector-major r x N, global).  Returns r (every thread).  Shared by k_svd_eig (N <= 512, one CTA
// for everything) and k_svd_vec (N > 512, after the grid-wide reduction).
__device__ int svd_vectors(const double* d, const double* e, const double* e2, const double* lam, int N, double tnorm,
                           double tt_eps, int rcap, double* __restrict__ work, double* __restrict__ Y,
                           double* __restrict__ Z, double* B, double* Q, double* dots, double* pc, double* ps, int* ipq,
                           int* order, int* misc, double* red) {
  const int tid = threadIdx.x, T = blockDim.x, wid = tid >> 5, ln = tid & 31, NW = T >> 5;
  // ---- 3. the tail rule (R21) and the cap
  if (tid == 0) {
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
    r = max(1, min(r, min(rcap, N)));
    misc[0] = r;
  }
  __syncthreads();
  const int r = misc[0];
  // ---- 4. inverse iteration on T - lambda I (one thread per wanted eigenvector)
  if (tid < r) {
    const int k = tid;
    const double lm = lam[N - 1 - k];
    double* dl = work + (int64_t)k * 6 * N;
    double* dd = dl + N;
    double* du = dd + N;
    double* du2 = du + N;
    double* pv = du2 + N;
    double* b = pv + N;
    const double pivmin = fmax(1e-16 * tnorm, 1e-300);
    for (int i = 0; i < N; ++i) {
      dd[i] = d[i] - lm;
      dl[i] = e[i];
      du[i] = e[i];
      du2[i] = 0.0;
      b[i] = start_value(i, k);
    }
    for (int i = 0; i + 1 < N; ++i) {
      if (fabs(dd[i]) >= fabs(dl[i])) {
        if (fabs(dd[i]) < pivmin) dd[i] = dd[i] < 0.0 ? -pivmin : pivmin;
        const double f = dl[i] / dd[i];
        dl[i] = f;
        dd[i + 1] -= f * du[i];
        pv[i] = 0.0;
      } else {
        const double f = dd[i] / dl[i];
        dd[i] = dl[i];
        dl[i] = f;
        const double t = du[i];
        du[i] = dd[i + 1];
        dd[i + 1] = t - f * dd[i + 1];
        if (i + 2 < N) {
          du2[i] = du[i + 1];
          du[i + 1] = -f * du[i + 1];
        }
        pv[i] = 1.0;
      }
    }
    if (fabs(dd[N - 1]) < pivmin) dd[N - 1] = dd[N - 1] < 0.0 ? -pivmin : pivmin;
    for (int it = 0; it < 3; ++it) {
      for (int i = 0; i + 1 < N; ++i) {
        if (pv[i] == 0.0) {
          b[i + 1] -= dl[i] * b[i];
        } else {
          const double t = b[i];
          b[i] = b[i + 1];
          b[i + 1] = t - dl[i] * b[i];
        }
      }
      b[N - 1] /= dd[N - 1];
      if (N >= 2) b[N - 2] = (b[N - 2] - du[N - 2] * b[N - 1]) / dd[N - 2];
      for (int i = N - 3; i >= 0; --i) b[i] = (b[i] - du[i] * b[i + 1] - du2[i] * b[i + 2]) / dd[i];
      double mx = 0.0;
      for (int i = 0; i < N; ++i) mx = fmax(mx, fabs(b[i]));
      const double s = mx > 0.0 ? 1.0 / mx : 1.0;
      for (int i = 0; i < N; ++i) b[i] *= s;
    }
    for (int i = 0; i < N; ++i) Y[(int64_t)k * N + i] = b[i];
  }
  __syncthreads();
  // ---- 5. CGS2 orthonormalisation (clusters of close eigenvalues give nearly parallel vectors)
  for (int k = 0; k < r; ++k) {
    double* yk = Y + (int64_t)k * N;
    for (int pass = 0; pass < 2; ++pass) {
      for (int j = wid; j < k; j += NW) {
        const double* yj = Y + (int64_t)j * N;
        double s = 0.0;
        for (int i = ln; i < N; i += 32) s += yk[i] * yj[i];
        s = warp_sum(s);
        if (ln == 0) dots[j] = s;
      }
      __syncthreads();
      for (int i = tid; i < N; i += T) {
        double v = yk[i];
        for (int j = 0; j < k; ++j) v -= dots[j] * Y[(int64_t)j * N + i];
        yk[i] = v;
      }
      __syncthreads();
    }
    double s2 = 0.0;
    for (int i = tid; i < N; i += T) s2 += yk[i] * yk[i];
    const double nrm = sqrt(blk_sum(s2, red));
    const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
    for (int i = tid; i < N; i += T) yk[i] *= inv;
    __syncthreads();
  }
  // ---- 6. Rayleigh-Ritz: B = Y^T T Y (T Y into Z as scratch)
  for (int q = tid; q < r * N; q += T) {
    const int k = q / N, i = q - k * N;
    const double* yk = Y + (int64_t)k * N;
    double v = d[i] * yk[i];
    if (i > 0) v += e[i - 1] * yk[i - 1];
    if (i + 1 < N) v += e[i] * yk[i + 1];
    Z[(int64_t)k * N + i] = v;
  }
  __syncthreads();
  for (int pq = wid; pq < r * r; pq += NW) {
    const int k = pq / r, l = pq - k * r;
    if (l < k) continue;
    double s = 0.0;
    for (int i = ln; i < N; i += 32) s += Y[(int64_t)k * N + i] * Z[(int64_t)l * N + i];
    s = warp_sum(s);
    if (ln == 0) {
      B[k * (RMAX + 1) + l] = s;
      B[l * (RMAX + 1) + k] = s;
    }
  }
  for (int q = tid; q < RMAX * (RMAX + 1); q += T) Q[q] = 0.0;
  __syncthreads();
  for (int k = tid; k < r; k += T) Q[k * (RMAX + 1) + k] = 1.0;
  __syncthreads();
  // ---- 7. parallel cyclic Jacobi on B (r x r): B <- J^T B J, Q <- Q J
  const int re = r + (r & 1), np = re / 2;
  for (int sweep = 0; sweep < 40 && r > 1; ++sweep) {
    double off = 0.0, fro = 0.0;
    for (int q = tid; q < r * r; q += T) {
      const int k = q / r, l = q - k * r;
      const double v = B[k * (RMAX + 1) + l];
      fro += v * v;
      if (k != l) off += v * v;
    }
    off = blk_sum(off, red);
    fro = blk_sum(fro, red);
    if (off <= 1e-32 * fro || fro == 0.0) break;
    for (int rd = 0; rd < re - 1; ++rd) {
      if (tid < np) {
        int p, q;
        if (tid == 0) {
          p = rd;
          q = re - 1;
        } else {
          p = (rd + tid) % (re - 1);
          q = (rd - tid + re - 1) % (re - 1);
        }
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double c = 1.0, s = 0.0;
        if (q < r) {
          const double apq = B[p * (RMAX + 1) + q];
          if (fabs(apq) > 1e-300) {
            const double th = (B[q * (RMAX + 1) + q] - B[p * (RMAX + 1) + p]) / (2.0 * apq);
            const double t = fabs(th) > 1e150 ? 0.5 / th : (th >= 0.0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
            c = 1.0 / sqrt(t * t + 1.0);
            s = t * c;
          }
        }
        ipq[2 * tid] = p;
        ipq[2 * tid + 1] = q;
        pc[tid] = c;
        ps[tid] = s;
      }
      __syncthreads();
      for (int it = tid; it < r * np; it += T) {  // columns: B J, Q J
        const int row = it / np, pr = it - row * np;
        const int p = ipq[2 * pr], q = ipq[2 * pr + 1];
        const double c = pc[pr], s = ps[pr];
        if (q < r && s != 0.0) {
          const double a = B[row * (RMAX + 1) + p], b = B[row * (RMAX + 1) + q];
          B[row * (RMAX + 1) + p] = c * a - s * b;
          B[row * (RMAX + 1) + q] = s * a + c * b;
          const double qa = Q[row * (RMAX + 1) + p], qb = Q[row * (RMAX + 1) + q];
          Q[row * (RMAX + 1) + p] = c * qa - s * qb;
          Q[row * (RMAX + 1) + q] = s * qa + c * qb;
        }
      }
      __syncthreads();
      for (int it = tid; it < r * np; it += T) {  // rows: J^T (B J)
        const int pr = it / r, col = it - pr * r;
        const int p = ipq[2 * pr], q = ipq[2 * pr + 1];
        const double c = pc[pr], s = ps[pr];
        if (q < r && s != 0.0) {
          const double a = B[p * (RMAX + 1) + col], b = B[q * (RMAX + 1) + col];
          B[p * (RMAX + 1) + col] = c * a - s * b;
          B[q * (RMAX + 1) + col] = s * a + c * b;
        }
      }
      __syncthreads();
    }
  }
  // ---- 8. Ritz values descending (ties: lower index first)
  if (tid < r) {
    const double v = B[tid * (RMAX + 1) + tid];
    int pos = 0;
    for (int l = 0; l < r; ++l) {
      const double w = B[l * (RMAX + 1) + l];
      if (w > v || (w == v && l < tid)) ++pos;
    }
    order[pos] = tid;
  }
  __syncthreads();
  // ---- 9. Z = Y Q (sorted), then 10. u = H_0 ... H_{N-3} z, one warp per vector
  for (int q = tid; q < r * N; q += T) {
    const int k = q / N, i = q - k * N;
    const int src = order[k];
    double v = 0.0;
    for (int l = 0; l < r; ++l) v += Y[(int64_t)l * N + i] * Q[l * (RMAX + 1) + src];
    Z[(int64_t)k * N + i] = v;
  }
  __syncthreads();
  return r;
}

// C: N x N symmetric (destroyed).  Vh: N x N (reflectors).  vg, pg: N.  work: 6 N RMAX.
// Y, Z: N RMAX each (vector-major).  Outputs: eig_asc[N] (all eigenvalues, bisection),
// lam[r] (Ritz values, descending), rank_out[0] = r, U[N x r] row-major (eigenvectors).
__global__ void __launch_bounds__(ST)
k_svd_eig(double* __restrict__ C, int N, double* __restrict__ Vh, double* __restrict__ vg, double* __restrict__ pg,
          double* __restrict__ work, double* __restrict__ Y, double* __restrict__ Z, double tt_eps, int rcap,
          double* __restrict__ eig_asc, double* __restrict__ lam_out, int* __restrict__ rank_out,
          double* __restrict__ U) {
  extern __shared__ double sm[];
  double* d = sm;                      // N
  double* e = d + N;                   // N
  double* e2 = e + N;                  // N
  double* lam = e2 + N;                // N
  vg = lam + N;                        // N: the Householder vector, in shared memory
  pg = vg + N;                         // N (the global vg / pg arguments are not used)
  double* red = pg + N;                // 40
  double* B = red + 40;                // RMAX x (RMAX + 1)
  double* Q = B + RMAX * (RMAX + 1);   // RMAX x (RMAX + 1)
  double* dots = Q + RMAX * (RMAX + 1);  // RMAX
  double* pc = dots + RMAX;            // RMAX / 2
  double* ps = pc + RMAX / 2;          // RMAX / 2
  int* ipq = reinterpret_cast<int*>(ps + RMAX / 2);  // RMAX (pairs) + RMAX (order) + 4
  int* order = ipq + RMAX;
  int* misc = order + RMAX;
  const int tid = threadIdx.x, T = blockDim.x, wid = tid >> 5, ln = tid & 31, NW = T >> 5;
  // ---- 1. Householder tridiagonalisation, H_k = I - 2 v v^T on indices k+1..N-1
  for (int k = 0; k + 2 < N; ++k) {
    const int L = N - k - 1;
    double* A = C + (int64_t)(k + 1) * N + (k + 1);
    double xs = 0.0;
    for (int i = tid; i < L; i += T) {
      const double xi = C[(int64_t)(k + 1 + i) * N + k];
      vg[i] = xi;
      xs += xi * xi;
    }
    const double nx2 = blk_sum(xs, red);
    const double x0 = vg[0];
    const double nx = sqrt(nx2);
    const double alpha = (x0 > 0.0) ? -nx : nx;
    const double nv2 = nx2 - 2.0 * alpha * x0 + alpha * alpha;
    if (tid == 0) {
      d[k] = C[(int64_t)k * N + k];
      e[k] = (nx2 > 0.0) ? alpha : 0.0;
    }
    if (nv2 <= 0.0 || nx2 == 0.0) {  // already reduced: identity reflector
      __syncthreads();
      if (tid == 0) e[k] = vg[0];
      for (int i = tid; i < L; i += T) Vh[(int64_t)k * N + i] = 0.0;
      __syncthreads();
      continue;
    }
    const double inv = 1.0 / sqrt(nv2);
    __syncthreads();
    for (int i = tid; i < L; i += T) {
      const double v = (i == 0 ? vg[0] - alpha : vg[i]) * inv;
      vg[i] = v;
      Vh[(int64_t)k * N + i] = v;
    }
    __syncthreads();
    for (int i = wid; i < L; i += NW) {
      double s = 0.0;
      for (int j = ln; j < L; j += 32) s += A[(int64_t)i * N + j] * vg[j];
      s = warp_sum(s);
      if (ln == 0) pg[i] = s;
    }
    __syncthreads();
    double kp = 0.0;
    for (int i = tid; i < L; i += T) kp += vg[i] * pg[i];
    const double K = blk_sum(kp, red);
    for (int i = tid; i < L; i += T) pg[i] = pg[i] - K * vg[i];
    __syncthreads();
    for (int q = tid; q < L * L; q += T) {
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
    e[N - 1] = 0.0;
  }
  __syncthreads();
  for (int i = tid; i < N; i += T) e2[i] = (i < N - 1) ? e[i] * e[i] : 0.0;
  // ---- 2. all eigenvalues by Sturm bisection (ascending)
  if (tid == 0) {
    double gl = 1e300, gu = -1e300;
    for (int i = 0; i < N; ++i) {
      const double rad = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < N ? fabs(e[i]) : 0.0);
      gl = fmin(gl, d[i] - rad);
      gu = fmax(gu, d[i] + rad);
    }
    red[0] = gl;
    red[1] = gu;
  }
  __syncthreads();
  const double gl = red[0], gu = red[1];
  const double span = fmax(gu - gl, 1e-300);
  const double tnorm = fmax(fabs(gl), fabs(gu));
  for (int i = tid; i < N; i += T) {
    double lo = gl - 1e-12 * span, hi = gu + 1e-12 * span;
    for (int it = 0; it < 200 && hi - lo > 1e-15 * fmax(fabs(lo), fabs(hi)) + 1e-300; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (sturm(d, e2, N, mid) <= i) lo = mid;
      else hi = mid;
    }
    lam[i] = fmax(0.5 * (lo + hi), 0.0);
  }
  __syncthreads();
  for (int i = tid; i < N; i += T) eig_asc[i] = lam[i];
  const int r = svd_vectors(d, e, e2, lam, N, tnorm, tt_eps, rcap, work, Y, Z, B, Q, dots, pc, ps, ipq, order, misc,
                          red);
  for (int k = wid; k < r; k += NW) {
    double* z = Z + (int64_t)k * N;
    for (int kk = N - 3; kk >= 0; --kk) {
      const int L = N - kk - 1;
      const double* v = Vh + (int64_t)kk * N;
      double s = 0.0;
      for (int i = ln; i < L; i += 32) s += v[i] * z[kk + 1 + i];
      s = warp_sum(s);
      for (int i = ln; i < L; i += 32) z[kk + 1 + i] -= 2.0 * s * v[i];
      __syncwarp();
    }
  }
  __syncthreads();
  for (int q = tid; q < r * N; q += T) {
    const int k = q / N, i = q - k * N;
    U[(int64_t)i * r + k] = Z[(int64_t)k * N + i];
  }
  if (tid < r) lam_out[tid] = fmax(B[order[tid] * (RMAX + 1) + order[tid]], 0.0);
  if (tid == 0) rank_out[0] = r;
}

// N > 512 (after launch_tridiag_eig): steps 3-9 in one CTA from the tridiagonal (d, e) and the
// ascending eigenvalues lam in global memory (copied to shared memory: 4 N + 2 RMAX (RMAX + 1)
// doubles <= 200 KB at N = 4096); eig_asc <- lam, lam_out (Ritz values, descending), rank_out.
__global__ void __launch_bounds__(ST)
k_svd_vec(const double* __restrict__ dg, const double* __restrict__ eg, const double* __restrict__ lamg, int N,
          double* __restrict__ work, double* __restrict__ Y, double* __restrict__ Z, double tt_eps, int rcap,
          double* __restrict__ eig_asc, double* __restrict__ lam_out, int* __restrict__ rank_out) {
  extern __shared__ double sm[];
  double* d = sm;                      // N
  double* e = d + N;                   // N
  double* e2 = e + N;                  // N
  double* lam = e2 + N;                // N
  double* red = lam + N;               // 40
  double* B = red + 40;                // RMAX x (RMAX + 1)
  double* Q = B + RMAX * (RMAX + 1);   // RMAX x (RMAX + 1)
  double* dots = Q + RMAX * (RMAX + 1);  // RMAX
  double* pc = dots + RMAX;            // RMAX / 2
  double* ps = pc + RMAX / 2;          // RMAX / 2
  int* ipq = reinterpret_cast<int*>(ps + RMAX / 2);
  int* order = ipq + RMAX;
  int* misc = order + RMAX;
  const int tid = threadIdx.x, T = blockDim.x;
  for (int i = tid; i < N; i += T) {
    d[i] = dg[i];
    e[i] = (i < N - 1) ? eg[i] : 0.0;
    lam[i] = lamg[i];
    eig_asc[i] = lamg[i];
  }
  __syncthreads();
  for (int i = tid; i < N; i += T) e2[i] = (i < N - 1) ? e[i] * e[i] : 0.0;
  if (tid == 0) {
    double gl = 1e300, gu = -1e300;
    for (int i = 0; i < N; ++i) {
      const double rad = (i > 0 ? fabs(e[i - 1]) : 0.0) + (i + 1 < N ? fabs(e[i]) : 0.0);
      gl = fmin(gl, d[i] - rad);
      gu = fmax(gu, d[i] + rad);
    }
    red[0] = fmax(fabs(gl), fabs(gu));
  }
  __syncthreads();
  const double tnorm = red[0];
  __syncthreads();
  const int r = svd_vectors(d, e, e2, lam, N, tnorm, tt_eps, rcap, work, Y, Z, B, Q, dots, pc, ps, ipq, order, misc,
                            red);
  if (tid < r) lam_out[tid] = fmax(B[order[tid] * (RMAX + 1) + order[tid]], 0.0);
  if (tid == 0) rank_out[0] = r;
}

// u = H_0 ... H_{N-3} z for every vector (one warp per vector; the 8 warps of a CTA read the same
// reflector rows, so L1 serves 7 of 8), U[N x r] row-major.  r from the device (rank_out).
__global__ void __launch_bounds__(256) k_backtransform(const double* __restrict__ Vh, int N,
                                                       const int* __restrict__ rank_in, double* __restrict__ Z,
                                                       double* __restrict__ U) {
  const int r = rank_in[0];
  const int k = blockIdx.x * 8 + (threadIdx.x >> 5), ln = threadIdx.x & 31;
  if (k >= r) return;
  double* z = Z + (int64_t)k * N;
  for (int kk = N - 3; kk >= 0; --kk) {
    const int L = N - kk - 1;
    const double* v = Vh + (int64_t)kk * N;
    double s = 0.0;
    for (int i = ln; i < L; i += 32) s += v[i] * z[kk + 1 + i];
    s = warp_sum(s);
    for (int i = ln; i < L; i += 32) z[kk + 1 + i] -= 2.0 * s * v[i];
    __syncwarp();
  }
  for (int i = ln; i < N; i += 32) U[(int64_t)i * r + k] = z[i];
}

// one CTA per column k of an fp64 rows x r matrix M: the sign that makes the largest-|.|
// entry positive (lowest index on ties); out (fp32, same layout) = sgn * M * scale[k]
// (scale nullable = 1; scale[k] = 0 gives a zero column), sgn[k] recorded
__global__ void __launch_bounds__(256) k_sign_cols(const double* __restrict__ M, int64_t rows, int r,
                                                   const double* __restrict__ scale, float* __restrict__ out,
                                                   double* __restrict__ sgn) {
  __shared__ double bv[8];
  __shared__ int64_t bi[8];
  const int k = blockIdx.x;
  const double sc = scale ? scale[k] : 1.0;
  double best = -1.0;
  int64_t bidx = 0;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) {
    const double a = fabs(M[i * r + k] * sc);
    if (a > best) {
      best = a;
      bidx = i;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bidx, o);
    if (ov > best || (ov == best && oi < bidx)) {
      best = ov;
      bidx = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    bv[threadIdx.x >> 5] = best;
    bi[threadIdx.x >> 5] = bidx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (bv[w] > best || (bv[w] == best && bi[w] < bidx)) {
        best = bv[w];
        bidx = bi[w];
      }
    bv[0] = (M[bidx * r + k] * sc < 0.0) ? -1.0 : 1.0;
    sgn[k] = bv[0];
  }
  __syncthreads();
  const double s = bv[0] * sc;
  for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) out[i * r + k] = (float)(M[i * r + k] * s);
}

// X'[k][j] = sum_s Spart[s][j][k] (fixed order): thread j reads its r contiguous doubles per
// split, writes row k coalesced across j
template <int R>
__global__ void k_rows_from_spart(const double* __restrict__ Spart, int nS, int64_t n, int r, float* __restrict__ Xn) {
  const int64_t nr = n * r;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    double acc[R];
#pragma unroll
    for (int k = 0; k < R; ++k) acc[k] = 0.0;
    for (int b = 0; b < nS; ++b) {
      const double* src = Spart + (int64_t)b * nr + j * r;
#pragma unroll
      for (int k = 0; k < R; ++k)
        if (k < r) acc[k] += src[k];
    }
#pragma unroll
    for (int k = 0; k < R; ++k)
      if (k < r) Xn[(int64_t)k * n + j] = (float)acc[k];
  }
}

// Vt[k][j] = V[j][k] (fp32, for the X V contraction); X'[k][j] = sgn_k s_k V[j][k] (after signs)
__global__ void k_v_rows(const double* __restrict__ V, int64_t n, int r, const double* __restrict__ mult,
                         const double* __restrict__ sgn, float* __restrict__ out) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n * r; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / n, j = t - k * n;
    double v = V[j * r + k];
    if (mult) v *= mult[k];
    if (sgn) v *= sgn[k];
    out[t] = (float)v;
  }
}

// s_k = sqrt(lambda_k), inv_k = 1 / s_k (0 for a non-positive or negligible eigenvalue)
__global__ void k_sing(const double* __restrict__ lam, int r, double* __restrict__ s, double* __restrict__ inv) {
  const int k = threadIdx.x;
  if (k < r) {
    const double l0 = lam[0], l = lam[k];
    const bool ok = l > 0.0 && l > 1e-28 * l0;
    s[k] = ok ? sqrt(l) : 0.0;
    inv[k] = ok ? 1.0 / sqrt(l) : 0.0;
  }
}

}  // namespace

size_t svd_eig_bytes(int64_t N) {
  return sizeof(double) * ((size_t)N * N + 2 * (size_t)N + 6 * (size_t)N * RMAX + 2 * (size_t)N * RMAX + N + RMAX +
                           (size_t)N * RMAX + 64) +
         1024;
}

cudaError_t launch_svd_eig(double* C, int N, char* ws, double tt_eps, int rcap, double* eig_asc, double* lam,
                           int* d_rank, double* U, int num_sms, cudaStream_t st) {
  if (N > kRankMaxN || rcap > RMAX) return cudaErrorInvalidValue;
  double* Vh = reinterpret_cast<double*>(ws);
  double* vg = Vh + (size_t)N * N;
  double* pg = vg + N;
  double* work = pg + N;
  double* Y = work + 6 * (size_t)N * RMAX;
  double* Z = Y + (size_t)N * RMAX;
  if (N > 512) {
    // the grid-wide reduction (reflectors into Vh) and multisection, then steps 3-9 in one CTA
    // and the back-transformation with a warp per vector.  d = vg, e and lam after Z.
    double* eg = Z + (size_t)N * RMAX;
    double* lamg = eg + N;
    unsigned* ctr = reinterpret_cast<unsigned*>(lamg + N);
    cudaError_t e = launch_tridiag_eig(C, N, pg, vg, eg, lamg, ctr, Vh, num_sms, st);
    if (e) return e;
    const size_t smv = sizeof(double) * (4 * (size_t)N + 40 + 2 * RMAX * (RMAX + 1) + RMAX + RMAX) +
                       sizeof(int) * (2 * RMAX + 8);
    e = smem_optin((const void*)(k_svd_vec), smv);
    if (e) return e;
    k_svd_vec<<<1, ST, smv, st>>>(vg, eg, lamg, N, work, Y, Z, tt_eps, rcap, eig_asc, lam, d_rank);
    if ((e = cudaGetLastError())) return e;
    k_backtransform<<<RMAX / 8, 256, 0, st>>>(Vh, N, d_rank, Z, U);
    return cudaGetLastError();
  }
  const size_t sm = sizeof(double) * (6 * (size_t)N + 40 + 2 * RMAX * (RMAX + 1) + RMAX + RMAX) + sizeof(int) * (2 * RMAX + 8);
  cudaError_t e = smem_optin((const void*)(k_svd_eig), sm);
  if (e) return e;
  k_svd_eig<<<1, ST, sm, st>>>(C, N, Vh, vg, pg, work, Y, Z, tt_eps, rcap, eig_asc, lam, d_rank, U);
  return cudaGetLastError();
}

cudaError_t launch_sign_cols(const double* M, int64_t rows, int r, const double* scale, float* out, double* sgn,
                             cudaStream_t st) {
  k_sign_cols<<<r, 256, 0, st>>>(M, rows, r, scale, out, sgn);
  return cudaGetLastError();
}

cudaError_t launch_rows_from_spart(const double* Spart, int nS, int64_t n, int r, float* Xn, cudaStream_t st) {
  const unsigned g = (unsigned)std::max<int64_t>(1, std::min<int64_t>(1184, (n + 127) / 128));
  if (r <= 8) k_rows_from_spart<8><<<g, 128, 0, st>>>(Spart, nS, n, r, Xn);
  else if (r <= 16) k_rows_from_spart<16><<<g, 128, 0, st>>>(Spart, nS, n, r, Xn);
  else if (r <= 32) k_rows_from_spart<32><<<g, 128, 0, st>>>(Spart, nS, n, r, Xn);
  else k_rows_from_spart<64><<<g, 128, 0, st>>>(Spart, nS, n, r, Xn);
  return cudaGetLastError();
}

cudaError_t launch_v_rows(const double* V, int64_t n, int r, const double* mult, const double* sgn, float* out,
                          cudaStream_t st) {
  const int64_t g = std::min<int64_t>(1184, (n * r + 255) / 256);
  k_v_rows<<<(unsigned)std::max<int64_t>(g, 1), 256, 0, st>>>(V, n, r, mult, sgn, out);
  return cudaGetLastError();
}

cudaError_t launch_sing(const double* lam, int r, double* s, double* inv, cudaStream_t st) {
  k_sing<<<1, 64, 0, st>>>(lam, r, s, inv);
  return cudaGetLastError();
}

}  // namespace ntt
