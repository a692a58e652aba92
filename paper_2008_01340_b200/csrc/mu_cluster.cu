// mu_cluster.cu -- "cluster mode" (SURVEY s.8(a) a6, s.8(d) tail rows): the whole MU loop of a
// mid-size unfolding (config 3 steps 4-5: 256 x 1024 and 256 x 32; config 4 steps 5-6:
// 30 x 7776, 30 x 1296) in ONE thread-block cluster of CS <= 16 CTAs, X resident in the
// cluster's distributed shared memory for all iterations.  CTA c of the cluster owns the
// columns [c n / CS, (c+1) n / CS) of X and H and the rows [c m / CS, (c+1) m / CS) of W.
//
// Per MU iteration (include/ntt.h ntt_nmf_mu; Alg. 4-6; readings R1-R4):
//   1. CTA c sums the rows it owns of P = X H^T, and all of Q = H H^T, over the CS published
//      per-CTA partials (DSMEM reads, fixed order c' = 0..CS-1), applies
//      W <- W o P / (W Q + eps) to those rows (fp64 quotient, rounded to fp32, as persist_step)
//      and forms its rows' part of G = W^T W (fp64)            -> cluster barrier
//   2. every CTA gathers the new W rows and the CS Gram parts (fixed order) over DSMEM
//   3. H <- H o (W^T X) / (G H + eps) on its own columns (fp32, as k_tiny), then the next
//      partials P_c = X_c Hn_c^T (fp32 inside 64-column blocks, fp64 across) and
//      Q_c = Hn_c Hn_c^T (fp32 within a warp's columns, fp64 across warps), published in its
//      shared memory                                           -> cluster barrier
// Two cluster barriers and no global-memory round trip per iteration (the persistent grid
// kernels pay two grid barriers, an L2 slice reduction and a redundant full W update).
// H is kept transposed in shared memory (HT[j][k]: one column's ranks are one broadcast
// 16-byte load); the rank loops use packed FFMA2.  Every sum runs in a fixed order, so results
// are deterministic.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace ntt {

namespace {

constexpr int CLU_T = 512;           // threads per CTA
constexpr int CLU_NW = CLU_T / 32;   // warps per CTA
constexpr int CLU_BLK = 64;          // fp32 column block of the P partials (fp64 across blocks)
constexpr int CLU_MAXCS = 16;

// r0(c) = first W row owned by cluster rank c; first column of rank c
// (cs is a power of two, c m and c n fit in 32 bits: n <= CLU_MAXCS * 4096)
__host__ __device__ inline int clu_row0(int c, int m, int lcs) { return (c * m) >> lcs; }
__host__ __device__ inline int clu_col0(int c, int n, int lcs) { return (c * n) >> lcs; }

}  // namespace

// geometry shared by the host plan and the kernel (passed by value)
struct CluPlan {
  int m, r, rk, cs, lcs;  // lcs = log2(cs)
  int n;
  int ncmax;     // max columns per CTA
  int ldc;       // smem row stride of X (odd: conflict-free column reads)
  int nq;        // row chunks of the S = W^T X partials (phase 3a)
  int nc2;       // column chunks of the P partials (phase 3b)
  int nch1;      // row chunks of the Gram part (phase 1)
  int rows_max;  // max W rows per CTA
  size_t oX, oH, oH2, oW, oS, oPQ, oCH, oQw, oPl, oWp, oGp, oGc, oGf, oOwn, bytes;
};

namespace {

template <int RK>
__global__ void __launch_bounds__(CLU_T, 1)
k_clu(const float* __restrict__ X, int64_t ldx, float* __restrict__ W, float* __restrict__ H, float eps, int iters,
      const CluPlan g, unsigned long long* trace) {
  // diagnostics (NTT_PERSIST_TRACE): CTA 0's globaltimer at 8 phase points of iterations < 512
  auto stamp = [&](int it, int k) {
    if (trace && threadIdx.x == 0 && blockIdx.x == 0 && it < 512) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      trace[12288 + it * 8 + k] = t;
    }
  };
  static_assert(CLU_T % RK == 0 && 32 % RK == 0, "rank class must divide the warp");
  constexpr int R2 = RK / 2, R4 = RK / 4;
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  const int CS = g.cs, m = g.m, r = g.r, ldc = g.ldc;
  const int tid = threadIdx.x, T = CLU_T, lane = tid & 31, warp = tid >> 5;
  extern __shared__ __align__(16) unsigned char sm[];
  float* Xs = reinterpret_cast<float*>(sm + g.oX);     // [m][ldc] own columns
  float* HT = reinterpret_cast<float*>(sm + g.oH);     // [ncmax][RK] H transposed (ranks >= r zero)
  float* HT2 = reinterpret_cast<float*>(sm + g.oH2);   // the other buffer of the H update
  float* Ws = reinterpret_cast<float*>(sm + g.oW);     // [m][RK] replicated W
  float* Sp = reinterpret_cast<float*>(sm + g.oS);     // [nq][ncmax][RK] S = W^T X row-chunk partials
  // P rows padded to LDP = RK + 2 doubles: the per-row 16-byte stores of consecutive rows by
  // consecutive lanes hit distinct bank groups (a 64-byte stride made every store 4x conflicted)
  constexpr int LDP = RK + 2;
  double* PQ = reinterpret_cast<double*>(sm + g.oPQ);  // published: P_c [m][LDP] | Q_c [RK][RK]
  double* CH = reinterpret_cast<double*>(sm + g.oCH);  // [nc2][m][LDP] column-chunk partials of P_c
  double* Qw = reinterpret_cast<double*>(sm + g.oQw);  // [NW][RK][RK] per-warp partials of Q_c
  double* Pl = reinterpret_cast<double*>(sm + g.oPl);  // owned rows of P [rows][RK] | Q [RK][RK]
  float* Wp = reinterpret_cast<float*>(sm + g.oWp);    // published: new W of the owned rows
  double* Gp = reinterpret_cast<double*>(sm + g.oGp);  // published: Gram part of the owned rows
  double* Gc = reinterpret_cast<double*>(sm + g.oGc);  // [nch1][RK][RK] Gram row-chunk partials
  float* Gf = reinterpret_cast<float*>(sm + g.oGf);    // [RK][RK] G (fp32, for E = G H)
  unsigned char* own = sm + g.oOwn;                    // [m] owning rank of each W row

  const int lcs = g.lcs;
  const int j0 = clu_col0(c, g.n, lcs), ncl = clu_col0(c + 1, g.n, lcs) - j0;
  const int r0 = clu_row0(c, m, lcs), nrow = clu_row0(c + 1, m, lcs) - r0;
  const int kk = tid % RK;  // this thread's rank in the (column, rank) phases (T % RK == 0)

  // ---- load the own column block of X, H (transposed) and all of W
  for (int64_t e = tid; e < (int64_t)m * ncl; e += T) {
    const int i = (int)(e / ncl), j = (int)(e % ncl);
    Xs[i * ldc + j] = X[(int64_t)i * ldx + j0 + j];
  }
  for (int e = tid; e < RK * ncl; e += T) {
    const int k = e / ncl, j = e % ncl;
    HT[j * RK + k] = k < r ? H[(int64_t)k * g.n + j0 + j] : 0.0f;
  }
  for (int e = tid; e < m * RK; e += T) {
    const int i = e / RK, k = e % RK;
    Ws[e] = k < r ? W[(int64_t)i * r + k] : 0.0f;
  }
  for (int o = 0; o < CS; ++o)
    for (int i = clu_row0(o, m, lcs) + tid; i < clu_row0(o + 1, m, lcs); i += T) own[i] = (unsigned char)o;
  __syncthreads();

  // ---- (column j, rank kk) items: optionally the H update (reads Sp, G row kk), and the
  //      warp's part of Q_c = Hn Hn^T (lane groups of RK lanes share a column; products in
  //      fp32 over the warp's columns, the warps' parts summed in fp64, fixed order)
  auto hupdate_q = [&](bool update, const float (&grow)[RK], const float* Hin, float* Hout) {
    float qa[RK];
#pragma unroll
    for (int l = 0; l < RK; ++l) qa[l] = 0.0f;
    const int rounds = (ncl * RK + T - 1) / T;  // uniform over the CTA (shuffles below)
    for (int rd = 0; rd < rounds; ++rd) {
      const int t = rd * T + tid;
      const int j = t / RK;
      float hn = 0.0f;
      if (j < ncl) {
        if (update) {
          float s = 0.0f;
          for (int q = 0; q < g.nq; ++q) s += Sp[((size_t)q * g.ncmax + j) * RK + kk];
          const float4* hp = reinterpret_cast<const float4*>(Hin + j * RK);
          float ek = 0.0f;
#pragma unroll
          for (int l4 = 0; l4 < R4; ++l4) {
            const float4 h4 = hp[l4];
            ek = fmaf(grow[4 * l4 + 0], h4.x, ek);
            ek = fmaf(grow[4 * l4 + 1], h4.y, ek);
            ek = fmaf(grow[4 * l4 + 2], h4.z, ek);
            ek = fmaf(grow[4 * l4 + 3], h4.w, ek);
          }
          hn = kk < r ? mu_quot(Hin[j * RK + kk], s, ek, eps) : 0.0f;
          Hout[j * RK + kk] = hn;
        } else {
          hn = Hin[j * RK + kk];
        }
      }
      const int base = lane & ~(RK - 1);
#pragma unroll
      for (int l = 0; l < RK; ++l) qa[l] = fmaf(hn, __shfl_sync(0xffffffffu, hn, base + l), qa[l]);
    }
#pragma unroll
    for (int o = RK; o < 32; o <<= 1)
#pragma unroll
      for (int l = 0; l < RK; ++l) qa[l] += __shfl_xor_sync(0xffffffffu, qa[l], o);
    if (lane < RK)
#pragma unroll
      for (int l = 0; l < RK; ++l) Qw[(warp * RK + lane) * RK + l] = (double)qa[l];
    __syncthreads();
    for (int e = tid; e < RK * RK; e += T) {
      double s = 0.0;
      for (int w = 0; w < CLU_NW; ++w) s += Qw[w * RK * RK + e];
      PQ[m * LDP + e] = s;
    }
  };

  // ---- P_c = X_c Hn_c^T: (row a, column chunk ch) items, all RK ranks per item (lanes run
  //      over consecutive rows: conflict-free X columns, broadcast H rows)
  auto pside = [&](const float* Hc) {
    constexpr int NR = RK == 8 ? 2 : 1;  // rows per item (two independent accumulator sets)
    const int nc2 = g.nc2, mh = (m + NR - 1) / NR;
    for (int t = tid; t < mh * nc2; t += T) {
      const int ap = t % mh, ch = t / mh;
      const float* av[NR];
#pragma unroll
      for (int u = 0; u < NR; ++u) av[u] = Xs + (ap + u * mh < m ? ap + u * mh : ap) * ldc;
      const int b0 = ncl * ch / nc2, b1 = ncl * (ch + 1) / nc2;
      double acc[NR][RK];
#pragma unroll
      for (int u = 0; u < NR; ++u)
#pragma unroll
        for (int k = 0; k < RK; ++k) acc[u][k] = 0.0;
      for (int jb = b0; jb < b1; jb += CLU_BLK) {
        const int je = min(b1, jb + CLU_BLK);
        float2 s[NR][R2];
#pragma unroll
        for (int u = 0; u < NR; ++u)
#pragma unroll
          for (int k = 0; k < R2; ++k) s[u][k] = make_float2(0.f, 0.f);
#pragma unroll 2
        for (int j = jb; j < je; ++j) {
          float2 x2[NR];
#pragma unroll
          for (int u = 0; u < NR; ++u) {
            const float x = av[u][j];
            x2[u] = make_float2(x, x);
          }
          const float4* hp = reinterpret_cast<const float4*>(Hc + j * RK);
#pragma unroll
          for (int l4 = 0; l4 < R4; ++l4) {
            const float4 h4 = hp[l4];
#pragma unroll
            for (int u = 0; u < NR; ++u) {
              s[u][2 * l4] = __ffma2_rn(x2[u], make_float2(h4.x, h4.y), s[u][2 * l4]);
              s[u][2 * l4 + 1] = __ffma2_rn(x2[u], make_float2(h4.z, h4.w), s[u][2 * l4 + 1]);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < NR; ++u)
#pragma unroll
          for (int k = 0; k < R2; ++k) {
            acc[u][2 * k] += (double)s[u][k].x;
            acc[u][2 * k + 1] += (double)s[u][k].y;
          }
      }
#pragma unroll
      for (int u = 0; u < NR; ++u) {
        const int a = ap + u * mh;
        if (a < m) {
          NTT_DCHECK(ch < nc2 && a < m);
          double* dst = nc2 == 1 ? PQ + a * LDP : CH + ((size_t)ch * m + a) * LDP;
#pragma unroll
          for (int k = 0; k < RK; k += 2)
            *reinterpret_cast<double2*>(dst + k) = make_double2(acc[u][k], acc[u][k + 1]);
        }
      }
    }
    if (nc2 > 1) {
      __syncthreads();
      for (int e = tid; e < m * RK; e += T) {
        double s = 0.0;
        const int pe = (e / RK) * LDP + e % RK;
        for (int ch = 0; ch < nc2; ++ch) s += CH[(size_t)ch * m * LDP + pe];
        PQ[pe] = s;
      }
    }
  };


  {
    float g0[RK] = {};
    hupdate_q(false, g0, HT, nullptr);
  }
  pside(HT);
  cl.sync();

  const int E1 = nrow * RK + RK * RK;
  for (int it = 0; it < iters; ++it) {
    stamp(it, 0);
    // ---- phase 1: owned rows of P and all of Q over the CS partials (fixed order, all of a
    //      thread's remote loads in flight together), W update of the owned rows
    for (int e = tid; e < E1; e += T) {
      const int off = e < nrow * RK ? (r0 + e / RK) * LDP + e % RK : m * LDP + (e - nrow * RK);
      NTT_DCHECK(off < m * LDP + RK * RK && e < g.rows_max * RK + RK * RK);
      double v[CLU_MAXCS];
#pragma unroll
      for (int q = 0; q < CLU_MAXCS; ++q) v[q] = q < CS ? cl.map_shared_rank(PQ, q)[off] : 0.0;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < CLU_MAXCS; ++q) s += v[q];
      Pl[e] = s;
    }
    __syncthreads();
    stamp(it, 1);
    const double* Ql = Pl + nrow * RK;
    for (int e = tid; e < nrow * RK; e += T) {
      const int i = e / RK, k = e % RK;
      float v = 0.0f;
      if (k < r) {
        const float* wr = Ws + (r0 + i) * RK;
        double d = 0.0;
#pragma unroll
        for (int l = 0; l < RK; ++l) d = fma((double)wr[l], Ql[l * RK + k], d);
        v = (float)mu_quot_fast((double)wr[k], Pl[e], d, (double)eps);
      }
      Wp[e] = v;
    }
    __syncthreads();
    stamp(it, 2);
    // Gram part of the owned rows: (entry, row chunk) items, chunks summed in order
    for (int t = tid; t < RK * RK * g.nch1; t += T) {
      const int kl = t % (RK * RK), ch = t / (RK * RK);
      const int k = kl / RK, l = kl % RK;
      const int i0 = nrow * ch / g.nch1, i1 = nrow * (ch + 1) / g.nch1;
      double s = 0.0;
      for (int i = i0; i < i1; ++i) s = fma((double)Wp[i * RK + k], (double)Wp[i * RK + l], s);
      Gc[t] = s;
    }
    __syncthreads();
    for (int kl = tid; kl < RK * RK; kl += T) {
      double s = 0.0;
      for (int ch = 0; ch < g.nch1; ++ch) s += Gc[ch * RK * RK + kl];
      Gp[kl] = s;
    }
    stamp(it, 3);
    cl.sync();  // B1: new W rows and Gram parts published
    stamp(it, 4);

    // ---- phase 2: gather W (all of a thread's remote loads in flight together) and G
    {
      constexpr int GW = 8;
      for (int e0 = 0; e0 < m * RK; e0 += GW * T) {
        float v[GW];
#pragma unroll
        for (int u = 0; u < GW; ++u) {
          const int e = e0 + u * T + tid;
          v[u] = 0.0f;
          if (e < m * RK) {
            const int i = e / RK, o = own[i];
            NTT_DCHECK(o < CS && i - clu_row0(o, m, lcs) < g.rows_max);
            v[u] = cl.map_shared_rank(Wp, o)[(i - clu_row0(o, m, lcs)) * RK + (e % RK)];
          }
        }
#pragma unroll
        for (int u = 0; u < GW; ++u) {
          const int e = e0 + u * T + tid;
          if (e < m * RK) Ws[e] = v[u];
        }
      }
    }
    // G = sum of the CS Gram parts (fixed order): one entry per thread, loads in flight together
    for (int kl = tid; kl < RK * RK; kl += T) {
      double v[CLU_MAXCS];
#pragma unroll
      for (int q = 0; q < CLU_MAXCS; ++q) v[q] = q < CS ? cl.map_shared_rank(Gp, q)[kl] : 0.0;
      double s = 0.0;
#pragma unroll
      for (int q = 0; q < CLU_MAXCS; ++q) s += v[q];
      Gf[kl] = ((kl / RK) < r && (kl % RK) < r) ? (float)s : 0.0f;
    }
    __syncthreads();
    stamp(it, 5);
    if (c == 0 && it == iters - 1)
      for (int e = tid; e < m * r; e += T) W[e] = Ws[(e / r) * RK + (e % r)];

    float grow[RK];  // row kk of G (fp32, for E = G H)
#pragma unroll
    for (int l = 0; l < RK; ++l) grow[l] = Gf[kk * RK + l];

    // ---- phase 3a: S = W^T X on (column pair (j, j + half), row chunk q) items into Sp
    {
      const int half = (ncl + 1) >> 1, nq = g.nq;
      for (int t = tid; t < half * nq; t += T) {
        const int ja = t % half, q = t / half;
        const bool two = ja + half < ncl;
        const int jb = two ? ja + half : ja;
        NTT_DCHECK(q < g.nq && jb < ncl && ncl <= g.ncmax);
        const int i0 = m * q / nq, i1 = m * (q + 1) / nq;
        float2 sa[R2], sb[R2];
#pragma unroll
        for (int k = 0; k < R2; ++k) sa[k] = sb[k] = make_float2(0.f, 0.f);
#pragma unroll 4
        for (int i = i0; i < i1; ++i) {
          const float xa = Xs[i * ldc + ja], xb = Xs[i * ldc + jb];
          const float2 xa2 = make_float2(xa, xa), xb2 = make_float2(xb, xb);
          const float4* wp = reinterpret_cast<const float4*>(Ws + i * RK);
#pragma unroll
          for (int l4 = 0; l4 < R4; ++l4) {
            const float4 w4 = wp[l4];
            const float2 wl = make_float2(w4.x, w4.y), wh = make_float2(w4.z, w4.w);
            sa[2 * l4] = __ffma2_rn(xa2, wl, sa[2 * l4]);
            sa[2 * l4 + 1] = __ffma2_rn(xa2, wh, sa[2 * l4 + 1]);
            sb[2 * l4] = __ffma2_rn(xb2, wl, sb[2 * l4]);
            sb[2 * l4 + 1] = __ffma2_rn(xb2, wh, sb[2 * l4 + 1]);
          }
        }
        float4* spa = reinterpret_cast<float4*>(Sp + ((size_t)q * g.ncmax + ja) * RK);
        float4* spb = reinterpret_cast<float4*>(Sp + ((size_t)q * g.ncmax + jb) * RK);
#pragma unroll
        for (int l4 = 0; l4 < R4; ++l4) {
          spa[l4] = make_float4(sa[2 * l4].x, sa[2 * l4].y, sa[2 * l4 + 1].x, sa[2 * l4 + 1].y);
          if (two) spb[l4] = make_float4(sb[2 * l4].x, sb[2 * l4].y, sb[2 * l4 + 1].x, sb[2 * l4 + 1].y);
        }
      }
    }
    __syncthreads();
    // ---- phase 3a': H update (HT -> HT2) and Q_c of the new H
    hupdate_q(true, grow, HT, HT2);
    {
      float* t2 = HT;
      HT = HT2;
      HT2 = t2;
    }
    __syncthreads();
    stamp(it, 6);
    if (it + 1 < iters) {
      pside(HT);
      stamp(it, 7);
      cl.sync();  // B2: P_c, Q_c published (and every gather of phase 2 done)
    }
  }
  for (int e = tid; e < r * ncl; e += T) {
    const int k = e / ncl, j = e % ncl;
    H[(int64_t)k * g.n + j0 + j] = HT[j * RK + k];
  }
  cl.sync();  // keep this CTA's shared memory alive until every DSMEM read of it is done
}

size_t al16(size_t v) { return (v + 15) & ~size_t(15); }

int max_smem() {
  static const int mx = [] {
    int d = 0, v = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, d);
    return v;
  }();
  return mx;
}

CluPlan make_plan(int64_t m, int64_t n, int r, int cs) {
  CluPlan g{};
  g.m = (int)m;
  g.n = (int)n;
  g.r = r;
  g.rk = r <= 8 ? 8 : 16;
  g.cs = cs;
  g.lcs = cs == 1 ? 0 : cs == 2 ? 1 : cs == 4 ? 2 : cs == 8 ? 3 : 4;
  const int RK = g.rk;
  g.ncmax = (int)((n + cs - 1) / cs);
  g.ldc = (g.ncmax & 1) ? g.ncmax : g.ncmax + 1;
  g.rows_max = (int)((m + cs - 1) / cs);
  // phase 3a: row chunks so that (column, chunk) items fill the CTA, >= 8 rows per chunk
  int nq = CLU_T / std::max((g.ncmax + 1) / 2, 1);
  nq = std::min<int>(nq, (int)std::max<int64_t>(1, m / 8));
  g.nq = std::max(1, nq);
  // phase 3b: column chunks so that (row, chunk) items fill the CTA, >= 16 columns per chunk
  int nc2 = CLU_T / (int)((m + (RK == 8 ? 1 : 0)) / (RK == 8 ? 2 : 1));
  nc2 = std::min(nc2, std::max(1, g.ncmax / 16));
  g.nc2 = std::max(1, nc2);
  int nch1 = CLU_T / (RK * RK);
  nch1 = std::min(nch1, std::max(1, g.rows_max / 4));
  g.nch1 = std::max(1, nch1);
  size_t o = 0;
  g.oX = o;
  o = al16(o + sizeof(float) * (size_t)m * g.ldc);
  g.oH = o;
  o = al16(o + sizeof(float) * (size_t)g.ncmax * RK);
  g.oH2 = o;
  o = al16(o + sizeof(float) * (size_t)g.ncmax * RK);
  g.oW = o;
  o = al16(o + sizeof(float) * (size_t)m * RK);
  g.oS = o;
  o = al16(o + sizeof(float) * (size_t)g.nq * g.ncmax * RK);
  g.oPQ = o;
  o = al16(o + sizeof(double) * (size_t)(m * (RK + 2) + RK * RK));
  g.oCH = o;
  if (g.nc2 > 1) o = al16(o + sizeof(double) * (size_t)g.nc2 * m * (RK + 2));
  g.oQw = o;
  o = al16(o + sizeof(double) * (size_t)CLU_NW * RK * RK);
  g.oPl = o;
  o = al16(o + sizeof(double) * (size_t)(g.rows_max * RK + RK * RK));
  g.oWp = o;
  o = al16(o + sizeof(float) * (size_t)g.rows_max * RK);
  g.oGp = o;
  o = al16(o + sizeof(double) * (size_t)RK * RK);
  g.oGc = o;
  o = al16(o + sizeof(double) * (size_t)g.nch1 * RK * RK);
  g.oGf = o;
  o = al16(o + sizeof(float) * (size_t)RK * RK);
  g.oOwn = o;
  o = al16(o + (size_t)m);
  g.bytes = o;
  return g;
}

template <int RK>
cudaError_t cluster_config(int cs, size_t smem) {
  cudaError_t e = smem_optin((const void*)k_clu<RK>, smem);
  if (e != cudaSuccess) return e;
  if (cs > 8) {
    e = cudaFuncSetAttribute(k_clu<RK>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// can a cluster of cs CTAs with smem bytes each be scheduled (cached per (RK, cs, smem band))
bool cluster_fits(int rk, int cs, size_t smem) {
  static std::mutex mu;
  static int cache[2][5][8];  // 0 unknown, 1 yes, 2 no; smem banded by 32 KB
  const int a = rk == 8 ? 0 : 1, b = cs == 1 ? 0 : cs == 2 ? 1 : cs == 4 ? 2 : cs == 8 ? 3 : 4;
  const int sb = (int)std::min<size_t>(7, smem / (32 * 1024));
  std::lock_guard<std::mutex> lk(mu);
  if (cache[a][b][sb]) return cache[a][b][sb] == 1;
  const size_t probe = std::min<size_t>((size_t)(sb + 1) * 32 * 1024, (size_t)max_smem() - 1024);
  cudaError_t e = rk == 8 ? cluster_config<8>(cs, probe) : cluster_config<16>(cs, probe);
  int ncl = 0;
  if (e == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs);
    cfg.blockDim = dim3(CLU_T);
    cfg.dynamicSmemBytes = probe;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    e = rk == 8 ? cudaOccupancyMaxActiveClusters(&ncl, k_clu<8>, &cfg)
                : cudaOccupancyMaxActiveClusters(&ncl, k_clu<16>, &cfg);
  }
  cudaGetLastError();  // a failed probe leaves no sticky error
  cache[a][b][sb] = (e == cudaSuccess && ncl > 0) ? 1 : 2;
  return cache[a][b][sb] == 1;
}

}  // namespace

// Cluster size for (m, n, r): the smallest power of two that leaves <= kCluEntries entries and
// <= kCluCols columns of X per CTA, raised until the shared-memory plan fits; 0 = not eligible
// (also for one CTA: 256 x 32 measured slower than the persistent kernel's 1-CTA grid).
int cluster_size_for(int64_t m, int64_t n, int r) {
  constexpr int64_t kCluEntries = 1024, kCluCols = 192;
  if (m < 1 || m > 255 + 1 || n < 1 || r < 1 || r > 16 || n > (int64_t)CLU_MAXCS * 4096) return 0;
  int cs = 1;
  while (cs < CLU_MAXCS && (m * ((n + cs - 1) / cs) > kCluEntries || (n + cs - 1) / cs > kCluCols)) cs *= 2;
  if ((n + cs - 1) / cs > kCluCols) return 0;  // measured: wide column blocks (30 x 7776) lose to the grid kernel
  if (const char* f = getenv("NTT_CLU_CS")) cs = std::max(cs, atoi(f));  // experiments: a larger cluster
  if (cs < 2) return 0;  // one CTA: the tiny / persistent kernels
  for (; cs <= CLU_MAXCS; cs *= 2) {
    const CluPlan g = make_plan(m, n, r, cs);
    if (g.bytes + 1024 <= (size_t)max_smem()) return cs;
  }
  return 0;
}

bool cluster_supported(int64_t m, int64_t n, int r) {
  const int cs = cluster_size_for(m, n, r);
  if (!cs) return false;
  const CluPlan g = make_plan(m, n, r, cs);
  return cluster_fits(g.rk, cs, g.bytes);
}

cudaError_t launch_cluster_mu(const float* X, int64_t ldx, int64_t m, int64_t n, int r, int iters, float eps, float* W,
                              float* H, cudaStream_t st, unsigned long long* trace) {
  const int cs = cluster_size_for(m, n, r);
  if (!cs || iters < 1) return cudaErrorInvalidValue;
  const CluPlan g = make_plan(m, n, r, cs);
  cudaError_t e = g.rk == 8 ? cluster_config<8>(cs, g.bytes) : cluster_config<16>(cs, g.bytes);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cs);
  cfg.blockDim = dim3(CLU_T);
  cfg.dynamicSmemBytes = g.bytes;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  if (g.rk == 8) return cudaLaunchKernelEx(&cfg, k_clu<8>, X, ldx, W, H, eps, iters, g, trace);
  return cudaLaunchKernelEx(&cfg, k_clu<16>, X, ldx, W, H, eps, iters, g, trace);
}

}  // namespace ntt
