// mu_small.cu -- 1-pass MU pass for unfoldings with very few rows (m <= 8; config 4's first
// step is 6 x 10 077 696 at r = 5, where H is 5/6 the size of X).  The warp-tile kernel of
// mu_fused.cu spends ~12 warp instructions per column on its 32-row tile machinery (TMA
// boxes, smem transposes, shuffles) at m = 6; here each lane owns two adjacent columns for
// the whole pass and keeps everything in registers:
//   x[i] = X[i][j..j+1] (float2, coalesced rows), h[k] = H[k][j..j+1]
//   update: S = W^T x, E = G h, Hn = h o S / (E + eps)     (FFMA2 over the column pair, R4)
//   acc:    P += x Hn^T, Q += Hn Hn^T in fp32 per lane over 16 rounds, then a fixed-order
//           fp64 warp butterfly into per-warp fp64 accumulators (R13), per-CTA partials
//           [grid][m r] / [grid][r r] for launch_wupdate2 (as launch_fused)
// Rounds are warp-uniform (lanes past n contribute zeros), so every sum has a fixed order.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ntt {

namespace {

constexpr int SMT = 256;   // threads per CTA
constexpr int SMW = SMT / 32;
constexpr int SCH = 16;    // rounds accumulated in fp32 before the fp64 flush

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  return make_float2(fmaf(a.x, b.x, c.x), fmaf(a.y, b.y, c.y));
}

template <int M, int R>
__global__ void __launch_bounds__(SMT, 2)
k_mu_small(const float* __restrict__ X, int64_t ldx, int m, int64_t n, int r, const float* __restrict__ W,
           const double* __restrict__ Gpart, int nG, float eps, float* __restrict__ H, double* __restrict__ Ppart,
           double* __restrict__ Qpart, int mode) {
  constexpr int NQ = R * (R + 1) / 2;
  constexpr int NA = M * R + NQ;
  __shared__ float Ws[M * R];
  __shared__ float Gs[R * R];
  __shared__ double accw[SMW][NA];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool upd = (mode & 1) != 0, acc = (mode & 2) != 0;
  for (int e = tid; e < M * R; e += SMT) {
    const int i = e / R, k = e % R;
    Ws[e] = (i < m && k < r) ? W[i * r + k] : 0.0f;
  }
  if (upd)
    for (int e = tid; e < R * R; e += SMT) {
      const int k = e / R, l = e % R;
      double s = 0.0;
      if (k < r && l < r)
        for (int b = 0; b < nG; ++b) s += Gpart[(int64_t)b * r * r + k * r + l];
      Gs[e] = (float)s;
    }
  for (int e = tid; e < SMW * NA; e += SMT) (&accw[0][0])[e] = 0.0;
  __syncthreads();

  float pa[M][R], qa[NQ];
#pragma unroll
  for (int i = 0; i < M; ++i)
#pragma unroll
    for (int k = 0; k < R; ++k) pa[i][k] = 0.0f;
#pragma unroll
  for (int q = 0; q < NQ; ++q) qa[q] = 0.0f;

  const int64_t npair = n >> 1;  // n % 4 == 0 (checked by the launcher)
  const int64_t twarps = (int64_t)gridDim.x * SMW;
  const int64_t gw = (int64_t)blockIdx.x * SMW + warp;
  const int64_t nround = (npair + twarps * 32 - 1) / (twarps * 32);
  auto flush = [&]() {
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      double v = a < M * R ? (double)pa[a / R][a % R] : (double)qa[a - M * R];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) accw[warp][a] += v;
    }
#pragma unroll
    for (int i = 0; i < M; ++i)
#pragma unroll
      for (int k = 0; k < R; ++k) pa[i][k] = 0.0f;
#pragma unroll
    for (int q = 0; q < NQ; ++q) qa[q] = 0.0f;
  };
  for (int64_t rd = 0; rd < nround; ++rd) {
    const int64_t p = (rd * twarps + gw) * 32 + lane;
    if (p < npair) {
      const int64_t j = 2 * p;
      float2 x[M], h[R];
#pragma unroll
      for (int i = 0; i < M; ++i)
        x[i] = (i < m) ? __ldcs(reinterpret_cast<const float2*>(X + (int64_t)i * ldx + j)) : make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < R; ++k)
        h[k] = (k < r) ? *reinterpret_cast<const float2*>(H + (int64_t)k * n + j) : make_float2(0.f, 0.f);
      if (upd) {
        float2 s[R], e[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
          s[k] = make_float2(0.f, 0.f);
          e[k] = make_float2(0.f, 0.f);
        }
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const float w = Ws[i * R + k];
            s[k] = ffma2(make_float2(w, w), x[i], s[k]);
          }
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int l = 0; l < R; ++l) {
            const float g = Gs[k * R + l];
            e[k] = ffma2(make_float2(g, g), h[l], e[k]);
          }
#pragma unroll
        for (int k = 0; k < R; ++k) {
          float2 hn;
          hn.x = __fdividef(__fmul_rn(h[k].x, s[k].x), __fadd_rn(e[k].x, eps));  // as the fused kernels (R4)
          hn.y = __fdividef(__fmul_rn(h[k].y, s[k].y), __fadd_rn(e[k].y, eps));
          if (k >= r) hn = make_float2(0.f, 0.f);
          if (k < r) *reinterpret_cast<float2*>(H + (int64_t)k * n + j) = hn;
          h[k] = hn;
        }
      }
      if (acc) {
#pragma unroll
        for (int i = 0; i < M; ++i)
#pragma unroll
          for (int k = 0; k < R; ++k) pa[i][k] = fmaf(x[i].y, h[k].y, fmaf(x[i].x, h[k].x, pa[i][k]));
        int q = 0;
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int l = 0; l <= k; ++l, ++q) qa[q] = fmaf(h[k].y, h[l].y, fmaf(h[k].x, h[l].x, qa[q]));
      }
    }
    if (acc && (rd % SCH == SCH - 1 || rd + 1 == nround)) flush();
  }
  if (!acc) return;
  __syncthreads();
  // fixed-order CTA reduction of the per-warp fp64 accumulators -> per-CTA partials
  for (int a = tid; a < NA; a += SMT) {
    double s = 0.0;
    for (int w = 0; w < SMW; ++w) s += accw[w][a];
    if (a < M * R) {
      const int i = a / R, k = a % R;
      if (i < m && k < r) Ppart[(int64_t)blockIdx.x * m * r + i * r + k] = s;
    } else {
      int q = a - M * R, k = 0;
      while (q > k) {
        q -= k + 1;
        ++k;
      }
      const int l = q;
      if (k < r && l < r) {
        Qpart[(int64_t)blockIdx.x * r * r + k * r + l] = s;
        Qpart[(int64_t)blockIdx.x * r * r + l * r + k] = s;
      }
    }
  }
}

template <int M, int R>
cudaError_t launch_small_t(const float* X, int64_t ldx, int m, int64_t n, int r, const float* W, const double* Gpart,
                           int nG, float eps, float* H, double* Ppart, double* Qpart, int mode, int grid,
                           cudaStream_t st) {
  k_mu_small<M, R><<<grid, SMT, 0, st>>>(X, ldx, m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode);
  return cudaGetLastError();
}

int small_rcls(int r) { return r <= 4 ? 4 : (r <= 6 ? 6 : 8); }
int small_mcls(int m) { return m <= 2 ? 2 : (m <= 4 ? 4 : (m <= 6 ? 6 : 8)); }

}  // namespace

bool small_supported(int64_t m, int64_t n, int r, int64_t ldx, const void* X, const void* H) {
  if (m < 1 || m > 8 || r < 1 || r > 8 || n < 4 || (n & 3) || (ldx & 1)) return false;
  if ((reinterpret_cast<uintptr_t>(X) & 7) || (reinterpret_cast<uintptr_t>(H) & 7)) return false;
  const int M = small_mcls((int)m), R = small_rcls(r);
  return M * R + R * (R + 1) / 2 <= 64;  // per-lane fp32 accumulators
}

// one wave: the kernels hold W and G in registers (up to ~250 of them), so 1 CTA of 256
// threads per SM for the larger classes; the partial count is the same for every class
int small_grid(int64_t n, int num_sms) {
  const int64_t need = (n / 2 + SMT - 1) / SMT;
  const int64_t g = need < 2 * num_sms ? need : 2 * num_sms;
  return (int)(g < 1 ? 1 : g);
}

cudaError_t launch_small(const float* X, int64_t ldx, int64_t m, int64_t n, int r, const float* W, const double* Gpart,
                         int nG, float eps, float* H, double* Ppart, double* Qpart, int mode, int grid,
                         cudaStream_t st) {
  const int M = small_mcls((int)m), R = small_rcls(r), mi = (int)m;
#define NTT_SMALL_CASE(MM, RR)                                                                                  \
  if (M == MM && R == RR)                                                                                       \
    return launch_small_t<MM, RR>(X, ldx, mi, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, st);
  NTT_SMALL_CASE(2, 4)
  NTT_SMALL_CASE(4, 4)
  NTT_SMALL_CASE(6, 4)
  NTT_SMALL_CASE(8, 4)
  NTT_SMALL_CASE(2, 6)
  NTT_SMALL_CASE(4, 6)
  NTT_SMALL_CASE(6, 6)
  NTT_SMALL_CASE(2, 8)
#undef NTT_SMALL_CASE
  return cudaErrorInvalidValue;
}

}  // namespace ntt
