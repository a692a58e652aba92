// mu_tiny.cu -- "tiny mode" (SURVEY s.8(a) a6, s.8(d) N8): the whole MU loop of a
// small unfolding (X of at most ~40k entries: config 1's steps, the tail steps of
// configs 3 and 4) in ONE CTA, with X, W, H and the r x r Grams resident in shared
// memory.  Per iteration (include/ntt.h ntt_nmf_mu, readings R1-R4):
//   P = X H^T, Q = H H^T         warp per row, fp32 per lane over 64 columns, fp64 across (R13)
//   W <- W o P / (W Q + eps)     fp64 quotient, rounded to fp32 (as k_wupdate)
//   G = W^T W                    fp64
//   H <- H o (W^T X) / (G H + eps)   per column, fp32 (as k_hpass)
// Every sum runs in a fixed order, so results are deterministic.  There is no
// launch, grid barrier or global round trip per iteration -- only CTA barriers.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace ntt {

namespace {

constexpr int TINY_THREADS = 512;
constexpr int TINY_BLK = 64;  // fp32 partial block: 32 lanes x 64 columns

// shared-memory row stride of X and H: odd, so that threads reading one column of
// consecutive rows hit distinct banks
__host__ __device__ inline int tiny_ld(int n) { return (n & 1) ? n : n + 1; }

template <int R>
struct TinyLayout {
  // offsets in bytes, all 16-aligned
  static size_t bytes(int m, int n, int nch) {
    const size_t ld = (size_t)tiny_ld(n);
    size_t o = 0;
    auto al = [](size_t v) { return (v + 15) & ~size_t(15); };
    o = al(o + sizeof(float) * (size_t)m * ld);       // X
    o = al(o + sizeof(float) * (size_t)R * ld);       // H (rows >= r zero)
    o = al(o + sizeof(float) * (size_t)m * R);        // W
    o = al(o + sizeof(float) * (size_t)m * R);        // W new
    o = al(o + sizeof(double) * (size_t)m * R);       // P
    o = al(o + sizeof(double) * (size_t)R * R);       // Q
    o = al(o + sizeof(float) * (size_t)R * R);        // G (fp32 for E = G H)
    o = al(o + sizeof(double) * (size_t)nch * (m * R + R * R));  // chunk partials (n <= 256)
    return o;
  }
};

template <int R>
__global__ void __launch_bounds__(TINY_THREADS, 1)
k_tiny(const float* __restrict__ X, int64_t ldx, int m, int n, int r, int iters, float eps, float* __restrict__ W,
       float* __restrict__ H, int nch, unsigned long long* trace) {
  auto stamp = [&](int it, int k) {  // diagnostics (NTT_PERSIST_TRACE): clock64 of thread 0
    if (trace && threadIdx.x == 0 && it < 512) trace[12288 + it * 8 + k] = (unsigned long long)clock64();
  };
  extern __shared__ __align__(16) unsigned char sm[];
  auto al = [](size_t v) { return (v + 15) & ~size_t(15); };
  const int ld = tiny_ld(n);
  size_t o = 0;
  float* Xs = reinterpret_cast<float*>(sm + o);
  o = al(o + sizeof(float) * (size_t)m * ld);
  float* Hs = reinterpret_cast<float*>(sm + o);
  o = al(o + sizeof(float) * (size_t)R * ld);
  float* Ws = reinterpret_cast<float*>(sm + o);
  o = al(o + sizeof(float) * (size_t)m * R);
  float* Wn = reinterpret_cast<float*>(sm + o);
  o = al(o + sizeof(float) * (size_t)m * R);
  double* P = reinterpret_cast<double*>(sm + o);
  o = al(o + sizeof(double) * (size_t)m * R);
  double* Q = reinterpret_cast<double*>(sm + o);
  o = al(o + sizeof(double) * (size_t)R * R);
  float* Gf = reinterpret_cast<float*>(sm + o);
  o = al(o + sizeof(float) * (size_t)R * R);
  double* part = reinterpret_cast<double*>(sm + o);
  o = al(o + sizeof(double) * (size_t)nch * (m * R + R * R));

  const int tid = threadIdx.x, T = blockDim.x;
  for (int64_t e = tid; e < (int64_t)m * n; e += T) {
    const int i = (int)(e / n), j = (int)(e % n);
    Xs[i * ld + j] = X[(int64_t)i * ldx + j];
  }
  for (int e = tid; e < R * n; e += T) {
    const int k = e / n, j = e % n;
    Hs[k * ld + j] = k < r ? H[(int64_t)k * n + j] : 0.0f;
  }
  for (int e = tid; e < m * R; e += T) {
    const int i = e / R, k = e % R;
    Ws[e] = k < r ? W[(int64_t)i * r + k] : 0.0f;
  }
  __syncthreads();

  const int EP = m * R, EQ = R * R, E = EP + EQ;
  const int nblk = (n + TINY_BLK - 1) / TINY_BLK;
  for (int it = 0; it < iters; ++it) {
    stamp(it, 0);
    if (n <= 256) {
    // ---- short rows: P = X H^T and Q = H H^T entry-parallel, entry e x chunk c of
    //      64-column blocks, fp32 inside a block, fp64 across.  P entries run row-fastest
    //      (e = k m + i: one X row per thread at a common column, H broadcast)
    for (int t = tid; t < E * nch; t += T) {
      const int e = t % E, c = t / E;
      const float* a;
      const float* bv;
      if (e < EP) {
        a = Xs + (e % m) * ld;
        bv = Hs + (e / m) * ld;
      } else {
        a = Hs + ((e - EP) / R) * ld;
        bv = Hs + ((e - EP) % R) * ld;
      }
      const int b0 = nblk * c / nch, b1 = nblk * (c + 1) / nch;
      double acc = 0.0;
      for (int bk = b0; bk < b1; ++bk) {
        const int j0 = bk * TINY_BLK, j1 = min(n, j0 + TINY_BLK);
        float s0 = 0.f, s1 = 0.f;
        int j = j0;
        for (; j + 1 < j1; j += 2) {
          s0 = fmaf(a[j], bv[j], s0);
          s1 = fmaf(a[j + 1], bv[j + 1], s1);
        }
        if (j < j1) s0 = fmaf(a[j], bv[j], s0);
        acc += (double)(s0 + s1);
      }
      part[c * E + e] = acc;
    }
    __syncthreads();
    stamp(it, 1);
    for (int e = tid; e < E; e += T) {
      double sv = 0.0;
      for (int c = 0; c < nch; ++c) sv += part[c * E + e];
      if (e < EP) P[(e % m) * R + e / m] = sv;
      else Q[e - EP] = sv;
    }
    __syncthreads();
    stamp(it, 2);
    } else {
    // ---- long rows: P = X H^T and Q = H H^T: one warp per row task (X row i, then H row k);
    //      lanes stride the columns (conflict-free), fp32 per lane over <= 64
    //      columns, fp64 across, fixed-order butterfly over the lanes
    {
      const int warp = tid >> 5, lane = tid & 31, nw = T >> 5;
      for (int task = warp; task < m + R; task += nw) {
        const float* a = task < m ? Xs + (int64_t)task * ld : Hs + (int64_t)(task - m) * ld;
        double acc[R];
#pragma unroll
        for (int k = 0; k < R; ++k) acc[k] = 0.0;
        for (int j0 = 0; j0 < n; j0 += 32 * TINY_BLK) {
          float s[R];
#pragma unroll
          for (int k = 0; k < R; ++k) s[k] = 0.0f;
          const int j1 = min(n, j0 + 32 * TINY_BLK);
          for (int j = j0 + lane; j < j1; j += 32) {
            const float x = a[j];
#pragma unroll
            for (int k = 0; k < R; ++k) s[k] = fmaf(x, Hs[k * ld + j], s[k]);
          }
#pragma unroll
          for (int k = 0; k < R; ++k) acc[k] += (double)s[k];
        }
#pragma unroll
        for (int k = 0; k < R; ++k) {
          double v = acc[k];
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
          acc[k] = v;
        }
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < R; ++k) {
            if (task < m) P[task * R + k] = acc[k];
            else Q[(task - m) * R + k] = acc[k];
          }
        }
      }
    }
    __syncthreads();
    }
    // ---- W update (fp64, R4)
    for (int e = tid; e < EP; e += T) {
      const int i = e / R, k = e % R;
      float v = 0.0f;
      if (k < r) {
        double d = 0.0;
        for (int l = 0; l < r; ++l) d += (double)Ws[i * R + l] * Q[l * R + k];
        v = (float)mu_quot((double)Ws[i * R + k], P[e], d, (double)eps);
      }
      Wn[e] = v;
    }
    __syncthreads();
    stamp(it, 3);
    for (int e = tid; e < EP; e += T) Ws[e] = Wn[e];
    // ---- G = W^T W (fp64, fixed order over rows)
    for (int e = tid; e < EQ; e += T) {
      const int k = e / R, l = e % R;
      double sg = 0.0;
      if (k < r && l < r)
        for (int i = 0; i < m; ++i) sg += (double)Wn[i * R + k] * (double)Wn[i * R + l];
      Gf[e] = (float)sg;
    }
    __syncthreads();
    stamp(it, 4);
    // ---- H update, one thread per column: S = W^T X[:, j], E = G H[:, j]
    for (int j = tid; j < n; j += T) {
      float s[R], h[R];
#pragma unroll
      for (int k = 0; k < R; ++k) {
        s[k] = 0.0f;
        h[k] = Hs[k * ld + j];
      }
      for (int i = 0; i < m; ++i) {
        const float x = Xs[i * ld + j];
#pragma unroll
        for (int k = 0; k < R; ++k) s[k] = fmaf(Ws[i * R + k], x, s[k]);
      }
#pragma unroll
      for (int k = 0; k < R; ++k) {
        float ek = 0.0f;
#pragma unroll
        for (int l = 0; l < R; ++l) ek = fmaf(Gf[k * R + l], h[l], ek);
        Hs[k * ld + j] = (k < r) ? mu_quot(h[k], s[k], ek, eps) : 0.0f;
      }
    }
    __syncthreads();
    stamp(it, 5);
  }
  for (int e = tid; e < r * n; e += T) H[e] = Hs[(e / n) * ld + e % n];
  for (int e = tid; e < m * r; e += T) W[e] = Ws[(e / r) * R + (e % r)];
}

int tiny_nch(int m, int r, int n) {
  const int R = r <= 4 ? 4 : (r <= 8 ? 8 : 16);
  const int E = m * R + R * R;
  int nch = TINY_THREADS / E;
  const int nblk = (n + TINY_BLK - 1) / TINY_BLK;
  if (nch > nblk) nch = nblk;
  return nch < 1 ? 1 : nch;
}

template <int R>
cudaError_t launch_tiny_t(const float* X, int64_t ldx, int m, int n, int r, int iters, float eps, float* W, float* H,
                          cudaStream_t st, unsigned long long* trace) {
  const int nch = tiny_nch(m, r, n);
  const size_t sm = TinyLayout<R>::bytes(m, n, nch);
  cudaError_t e = smem_optin((const void*)(k_tiny<R>), sm);
  if (e != cudaSuccess) return e;
  k_tiny<R><<<1, TINY_THREADS, sm, st>>>(X, ldx, m, n, r, iters, eps, W, H, nch, trace);
  return cudaGetLastError();
}

}  // namespace

// measured on B200: faster than the persistent fused kernel for m <= 64 (config 1,
// config 4 steps 7-9); config 3 step 5 (256 x 32) stays on the fused path
bool tiny_supported(int64_t m, int64_t n, int r) {
  if (r < 1 || r > 16 || m < 1 || n < 1 || m > 64) return false;
  const int R = r <= 4 ? 4 : (r <= 8 ? 8 : 16);
  if (m * n > 12 * 1024) return false;  // measured: the persistent fused kernel wins above (64 x 700, 30 x 1296)
  size_t b = R == 4 ? TinyLayout<4>::bytes((int)m, (int)n, tiny_nch((int)m, r, (int)n))
                    : (R == 8 ? TinyLayout<8>::bytes((int)m, (int)n, tiny_nch((int)m, r, (int)n))
                              : TinyLayout<16>::bytes((int)m, (int)n, tiny_nch((int)m, r, (int)n)));
  return b <= 220 * 1024;
}

cudaError_t launch_tiny(const float* X, int64_t ldx, int64_t m, int64_t n, int r, int iters, float eps, float* W,
                        float* H, cudaStream_t st, unsigned long long* trace) {
  if (r <= 4) return launch_tiny_t<4>(X, ldx, (int)m, (int)n, r, iters, eps, W, H, st, trace);
  if (r <= 8) return launch_tiny_t<8>(X, ldx, (int)m, (int)n, r, iters, eps, W, H, st, trace);
  return launch_tiny_t<16>(X, ldx, (int)m, (int)n, r, iters, eps, W, H, st, trace);
}

}  // namespace ntt
