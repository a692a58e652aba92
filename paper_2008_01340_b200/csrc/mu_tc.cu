// mu_tc.cu -- tensor-core (tcgen05, kind::tf32) 2-pass MU iteration for tall /
// square X (BASELINE configs 2 and 5: m x n = 4096 x 4096 r 16, 32768 x 65536
// r 32), where the contraction X H^T / W^T X is a real dense GEMM with a long K
// and FP32 FFMA cannot keep up with HBM (r/2 flop per byte, SURVEY s.0 #4).
//
// One MU iteration (include/ntt.h ntt_nmf_mu, readings R1-R4):
//   pass W   P = X Hcat^T          (Alg. 5 l.2)   k_skinny_tc<R, 0>
//   W update W <- W o P / (W Q + eps), G = W^T W  (Alg. 4)  k_tc_wupdate
//   pass H   S = X^T Wcat          (Alg. 6 l.2)   k_skinny_tc<R, 1>
//   H update H <- H o S / (G H + eps), Q = H H^T          k_tc_hupdate
//
// fp32 accuracy from TF32 tensor cores ("3xTF32"): every operand v is split
// v = hi + lo with hi = v truncated to TF32 (what the tensor core reads from a
// raw fp32 word) and lo = v - hi (exact in fp32); the products keep
// hi*hi + hi*lo + lo*hi and drop lo*lo (~2^-22 relative, SURVEY s.8(c) c.4:
// 3xTF32 drift 2.9e-7 vs the 1e-4 parity bar).  The MMA pair per K step is
//   D[:, 0:2R] (+)= A_hi * [B_hi | B_lo]      (N = 2R)
//   D[:, 0:R]  +=   A_lo *  B_hi              (TS, N = R)
// with A_hi the raw X tile in shared memory (pass W, SS form) or staged in TMEM
// (pass H, TS form), and A_lo always in TMEM: the converter warps read each X
// element once (LDS), split it, and store lo (and hi) with tcgen05.st.
// Measured on B200 (tools/tc_probe.cu): one M=128 K=8 tf32 MMA costs ~138
// cycles for any N in 8..128, so these passes are MMA-issue-bound at
// 2 MMAs per 128 x 8 X elements (<= ~15 B/clk/SM), not HBM-bound.  B = [B_hi | B_lo] is prepared by the update kernels
// (Hcat = [H; lo(H)] (2R x n), WcatT = [W^T; lo(W)^T] (2R x m)).
// The fp32 accumulator in TMEM is flushed to per-thread fp64 every
// `flush` K tiles (two-level sums, R13); split-K partials are fp64 and summed
// in fixed order by the update kernels (deterministic, R16).
//
// CTA = 10 warps, persistent (1 CTA / SM): warp 0 TMA producer, warp 1 MMA
// issuer (one thread), warps 2-5 converters, warps 6-9 epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"
#include "mu_tc.h"
#include "sm100.cuh"

namespace ntt {

namespace {
using namespace sm100;

constexpr int TC_BK = 32;     // K elements per stage (one 128-B swizzle row of fp32)
constexpr int TC_BM = 128;    // D rows per unit (UMMA M)
constexpr int TC_T = 4;       // TMEM A_lo buffers (32 columns each)
constexpr int TC_WARPS = 10;
constexpr int TC_THREADS = TC_WARPS * 32;
constexpr uint32_t TC_ABYTES = TC_BM * 128u;  // 16 KB A tile per stage

__device__ __forceinline__ float tf32_trunc(float v) { return __uint_as_float(__float_as_uint(v) & 0xFFFFE000u); }
__device__ __forceinline__ float tf32_lo(float v) { return __fsub_rn(v, tf32_trunc(v)); }

template <int R>
struct TcCfg {
  static constexpr int N1 = 2 * R;                        // [B_hi | B_lo]
  static constexpr uint32_t BBYTES = (uint32_t)N1 * 128u;  // B tile per stage
  static constexpr uint32_t SB = TC_ABYTES + BBYTES;
  static constexpr uint32_t TMEM_D = 0;                   // two accumulators of N1 columns
  static constexpr uint32_t TMEM_LO = 2 * N1;              // TC_T A_lo buffers of 32 columns
  static constexpr uint32_t TMEM_HI = TMEM_LO + TC_T * 32;  // TC_T A_hi buffers (MODE 1)
  static constexpr uint32_t TMEM_COLS = 512u;
};

// MODE 0: D (Mtot = m rows) = X * Hcat^T, A = X row block [128 rows][32 K] K-major.
// MODE 1: D (Mtot = n cols) = X^T * WcatT^T, A = X^T from four [32 K rows][32 M cols] boxes; the
//         converters stage both A_hi and A_lo in TMEM (an MN-major tf32 A read from shared
//         memory by the SS form gave wrong results on B200 in our probe, so it is not used).
// Units u = (mb, s): D rows [128 mb, 128 mb + 128), K tiles [s kchunk, (s+1) kchunk).
// part[(s * Mtot + row) * r + k] (fp64) for row < Mtot, k < r.
template <int R, int MODE>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_skinny_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t Mtot,
            int64_t ktiles, int nsplit, int64_t kchunk, int ns, int flush, int r, double* __restrict__ part,
            int evict_first) {
  using C = TcCfg<R>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)ns * C::SB);
  uint64_t* empty = full + ns;
  uint64_t* lo_full = empty + ns;
  uint64_t* lo_empty = lo_full + TC_T;
  uint64_t* acc_full = lo_empty + TC_T;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    tmem_alloc(tmem_slot, C::TMEM_COLS);
  } else if (warp == 1 && lane == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int t = 0; t < TC_T; ++t) {
      mbar_init(&lo_full[t], 4);
      mbar_init(&lo_empty[t], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 4);
    }
    fence_barrier_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  const int64_t nmb = (Mtot + TC_BM - 1) / TC_BM;
  const int64_t nunits = nmb * nsplit;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      const uint64_t pol = evict_first ? policy_evict_first() : policy_evict_normal();
      const uint64_t polB = policy_evict_normal();
      int s = 0;
      uint32_t ph = 0;  // ring position, incremental (no 64-bit division per stage)
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int64_t mb = u / nsplit, sp = u % nsplit;
        const int64_t k0 = sp * kchunk, k1 = ((k0 + kchunk < ktiles) ? k0 + kchunk : ktiles);
        for (int64_t kt = k0; kt < k1; ++kt, s = (s + 1 == ns) ? 0 : s + 1, ph ^= (s == 0) ? 1u : 0u) {
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_expect_tx(&full[s], C::SB);
          unsigned char* st = smem + (size_t)s * C::SB;
          if (MODE == 0) {
            tma_load_2d(st, &tmA, (int)(kt * TC_BK), (int)(mb * TC_BM), &full[s], pol);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tma_load_2d(st + q * 4096, &tmA, (int)(mb * TC_BM + 32 * q), (int)(kt * TC_BK), &full[s], pol);
          }
          tma_load_2d(st + TC_ABYTES, &tmB, (int)(kt * TC_BK), 0, &full[s], polB);
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      constexpr uint32_t id1 = idesc_tf32(TC_BM, C::N1, false, false);
      constexpr uint32_t id2 = idesc_tf32(TC_BM, R, false, false);
      int64_t g = 0;
      int s = 0, t = 0;
      uint32_t ph = 0, pht = 0;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int64_t sp = u % nsplit;
        const int64_t k0 = sp * kchunk, k1 = ((k0 + kchunk < ktiles) ? k0 + kchunk : ktiles);
        for (int64_t kt = k0; kt < k1; ++kt, s = (s + 1 == ns) ? 0 : s + 1, ph ^= (s == 0) ? 1u : 0u,
                     t = (t + 1) & (TC_T - 1), pht ^= (t == 0) ? 1u : 0u) {
          const int64_t i = kt - k0;  // tile index within the unit
          const bool gfirst = (i % flush) == 0;
          const bool glast = ((i + 1) % flush) == 0 || kt + 1 == k1;
          const int a = (int)(g & 1);
          if (gfirst) {
            mbar_wait(&acc_empty[a], (uint32_t)(((g >> 1) & 1) ^ 1));
            tc_fence_after();
          }
          mbar_wait(&full[s], ph);
          mbar_wait(&lo_full[t], pht);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + (size_t)s * C::SB);
          const uint32_t sb = sa + TC_ABYTES;
          const uint32_t dcol = tbase + C::TMEM_D + (uint32_t)a * C::N1;
#pragma unroll
          for (int kk = 0; kk < TC_BK / 8; ++kk) {
            const uint64_t bdesc = umma_desc_sw128(sb + kk * 32, 16, 1024);
            if (MODE == 0)  // A_hi = the raw X tile in shared memory (K-major)
              mma_tf32_ss(dcol, umma_desc_sw128(sa + kk * 32, 16, 1024), bdesc, id1, (gfirst && kk == 0) ? 0u : 1u);
            else            // A_hi = X^T staged in TMEM by the converters
              mma_tf32_ts(dcol, tbase + C::TMEM_HI + (uint32_t)t * 32 + kk * 8, bdesc, id1, (gfirst && kk == 0) ? 0u : 1u);
            mma_tf32_ts(dcol, tbase + C::TMEM_LO + (uint32_t)t * 32 + kk * 8, bdesc, id2, 1u);
          }
          mma_commit(&empty[s]);
          mma_commit(&lo_empty[t]);
          if (glast) {
            mma_commit(&acc_full[a]);
            ++g;
          }
        }
      }
    }
  } else if (warp < 6) {
    // ======================= converters: A_lo -> TMEM =======================
    const int q = warp & 3;  // TMEM lane quadrant this warp may access
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    int s = 0, t = 0;
    uint32_t ph = 0, pht = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int64_t sp = u % nsplit;
      const int64_t k0 = sp * kchunk, k1 = ((k0 + kchunk < ktiles) ? k0 + kchunk : ktiles);
      for (int64_t kt = k0; kt < k1; ++kt, s = (s + 1 == ns) ? 0 : s + 1, ph ^= (s == 0) ? 1u : 0u,
                   t = (t + 1) & (TC_T - 1), pht ^= (t == 0) ? 1u : 0u) {
        mbar_wait(&full[s], ph);
        mbar_wait(&lo_empty[t], pht ^ 1u);
        tc_fence_after();
        const unsigned char* st = smem + (size_t)s * C::SB;
        uint32_t v[32];
        if (MODE == 0) {
          // row rho = 32 q + lane of the [128][32] K-major tile
          const int rho = 32 * q + lane;
          const unsigned char* row = st + rho * 128;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const float4 x = *reinterpret_cast<const float4*>(row + ((ch ^ (rho & 7)) << 4));
            v[4 * ch + 0] = __float_as_uint(tf32_lo(x.x));
            v[4 * ch + 1] = __float_as_uint(tf32_lo(x.y));
            v[4 * ch + 2] = __float_as_uint(tf32_lo(x.z));
            v[4 * ch + 3] = __float_as_uint(tf32_lo(x.w));
          }
        } else {
          // column c = lane of box q ([32 K rows][32 cols]); K index = row i
          const unsigned char* box = st + q * 4096 + (lane & 3) * 4;
          const int chk = lane >> 2;
          uint32_t vh[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float x = *reinterpret_cast<const float*>(box + i * 128 + ((chk ^ (i & 7)) << 4));
            vh[i] = __float_as_uint(x);
            v[i] = __float_as_uint(tf32_lo(x));
          }
          tmem_st32(tbase + C::TMEM_HI + (uint32_t)t * 32 + lane_off, vh);
        }
        tmem_st32(tbase + C::TMEM_LO + (uint32_t)t * 32 + lane_off, v);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&lo_full[t]);
      }
    }
  } else {
    // ======================= epilogue: TMEM -> fp64 partials =======================
    const int q = warp & 3;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    int64_t g = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int64_t mb = u / nsplit, sp = u % nsplit;
      const int64_t k0 = sp * kchunk, k1 = ((k0 + kchunk < ktiles) ? k0 + kchunk : ktiles);
      const int64_t ngr = (k1 - k0 + flush - 1) / flush;
      double acc[R];
#pragma unroll
      for (int k = 0; k < R; ++k) acc[k] = 0.0;
      for (int64_t gi = 0; gi < ngr; ++gi, ++g) {
        const int a = (int)(g & 1);
        mbar_wait(&acc_full[a], (uint32_t)((g >> 1) & 1));
        tc_fence_after();
        const uint32_t d = tbase + C::TMEM_D + (uint32_t)a * C::N1 + lane_off;
#pragma unroll
        for (int c0 = 0; c0 < R; c0 += 16) {
          uint32_t hi[16], lo[16];
          tmem_ld16(d + c0, hi);
          tmem_ld16(d + R + c0, lo);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; ++k) acc[c0 + k] += (double)__uint_as_float(hi[k]) + (double)__uint_as_float(lo[k]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[a]);
      }
      const int64_t row = mb * TC_BM + 32 * q + lane;
      if (row < Mtot) {
        double* dst = part + ((int64_t)sp * Mtot + row) * r;
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (k < r) dst[k] = acc[k];
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tbase, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------- updates ---
// Both update kernels work on blocks of UPD_B rows (W) / columns (H) with 4 threads per row /
// column, each owning ranks k = kq + 4u: the per-thread serial work (the latency that bounds
// these small kernels: ~3 k warp instructions at 9.5 cycles each with one thread per row, ncu on
// config 2) is a quarter, and config 2's 4096 rows / columns give 128 CTAs instead of 32.
constexpr int UPD_THREADS = 128;
constexpr int UPD_B = 32;

// W update for UPD_B rows per CTA: P = sum_s Ppart[s] (fixed order), Q (r x r, reduced),
// W <- W o P / (W Q + eps) in fp64 (as k_wupdate), WcatT rows k < r: hi = Wn, rows R + k:
// lo(Wn); Gpart[cta] = Wn^T Wn over the CTA's rows.
template <int R>
__global__ void __launch_bounds__(UPD_THREADS)
k_tc_wupdate(float* __restrict__ W, int64_t m, int r, const double* __restrict__ Ppart, int nP,
             const double* __restrict__ Qred, float eps, float* __restrict__ WcatT, int64_t ldw,
             double* __restrict__ Gpart, unsigned* __restrict__ maxw) {
  constexpr int U = R / 4;
  __shared__ double Qs[R * R];
  __shared__ double Ps[UPD_B * R];
  __shared__ float Wo[UPD_B][R + 1];
  __shared__ float Wn[UPD_B][R + 1];
  const int tid = threadIdx.x;
  const int rr = r * r;
  const int64_t i0 = (int64_t)blockIdx.x * UPD_B;
  const int rows = (int)min((int64_t)UPD_B, m - i0);
  for (int t = tid; t < R * R; t += UPD_THREADS) {
    const int k = t / R, l = t % R;
    Qs[t] = (k < r && l < r) ? Qred[k * r + l] : 0.0;
  }
  for (int e = tid; e < UPD_B * R; e += UPD_THREADS) {
    const int row = e / R, k = e % R;
    Wo[row][k] = (row < rows && k < r) ? W[(i0 + row) * r + k] : 0.0f;
  }
  {
    // the block's rows are a contiguous run of rows * r doubles in every split partial:
    // element e = tid + 128 q, fp64 sums in registers, each split's loads issued together
    const int len = rows * r;
    const int64_t mr = m * r;
    double acc[U];
#pragma unroll
    for (int q = 0; q < U; ++q) acc[q] = 0.0;
    for (int b = 0; b < nP; ++b) {
      const double* src = Ppart + (int64_t)b * mr + i0 * r;
      double v[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int e = tid + q * UPD_THREADS;
        v[q] = e < len ? __ldcg(src + e) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < U; ++q) acc[q] += v[q];
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int e = tid + q * UPD_THREADS;
      if (e < len) Ps[(e / r) * R + e % r] = acc[q];
    }
  }
  __syncthreads();
  float wmax = 0.0f;
  {
    const int row = tid >> 2, kq = tid & 3;
    double d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) d[u] = 0.0;
#pragma unroll
    for (int l = 0; l < R; ++l) {
      const double wl = (double)Wo[row][l];
#pragma unroll
      for (int u = 0; u < U; ++u) d[u] = fma(wl, Qs[l * R + kq + 4 * u], d[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = kq + 4 * u;
      float wn = 0.0f;
      if (row < rows && k < r) wn = (float)mu_quot((double)Wo[row][k], Ps[row * R + k], d[u], (double)eps);
      Wn[row][k] = wn;
      wmax = fmaxf(wmax, wn);
    }
  }
  __syncthreads();
  for (int e = tid; e < rows * r; e += UPD_THREADS) W[i0 * r + e] = Wn[e / r][e % r];
  if (maxw) {  // max |W| for the fp16x2 scale (fp16 variant); order-independent
    for (int o = 16; o > 0; o >>= 1) wmax = fmaxf(wmax, __shfl_xor_sync(0xffffffffu, wmax, o));
    if ((tid & 31) == 0) atomicMax(maxw, __float_as_uint(wmax));
  }
  if (WcatT)
    for (int e = tid; e < R * UPD_B; e += UPD_THREADS) {
      const int k = e / UPD_B, row = e % UPD_B;
      if (row < rows) {
        const float v = Wn[row][k];
        WcatT[(int64_t)k * ldw + i0 + row] = v;
        WcatT[(int64_t)(R + k) * ldw + i0 + row] = tf32_lo(v);
      }
    }
  for (int t = tid; t < rr; t += UPD_THREADS) {
    const int k = t / r, l = t % r;
    double s0 = 0.0, s1 = 0.0;
    for (int q = 0; q < UPD_B; q += 2) {
      s0 = fma((double)Wn[q][k], (double)Wn[q][l], s0);
      s1 = fma((double)Wn[q + 1][k], (double)Wn[q + 1][l], s1);
    }
    Gpart[(int64_t)blockIdx.x * rr + t] = s0 + s1;
  }
}

// H update (or prep: update = false keeps H) for blocks of UPD_B columns (grid-stride):
// S = sum_s Spart[s][j] (fixed order), E = G H (fp32, G reduced in fp64),
// H <- H o S / (E + eps); Hcat rows k < r: hi = Hn, rows R + k: lo(Hn);
// Qpart[cta] = Hn Hn^T over the CTA's columns (fp64, in block order: deterministic).
template <int R>
__global__ void __launch_bounds__(UPD_THREADS)
k_tc_hupdate(float* __restrict__ H, int64_t n, int r, const double* __restrict__ Spart, int nS,
             const double* __restrict__ Gred, float eps, bool update, float* __restrict__ Hcat, int64_t ldh,
             double* __restrict__ Qpart, unsigned* __restrict__ maxh) {
  constexpr int U = R / 4;
  constexpr int NQ = (R * R + UPD_THREADS - 1) / UPD_THREADS;
  float hmax = 0.0f;
  __shared__ float Gs[R * R];
  __shared__ float Ho[R][UPD_B + 1];
  __shared__ float Hn[R][UPD_B + 1];
  __shared__ double Ss[UPD_B * R];
  const int tid = threadIdx.x;
  const int rr = r * r;
  if (update)
    for (int t = tid; t < R * R; t += UPD_THREADS) {
      const int k = t / R, l = t % R;
      Gs[t] = (k < r && l < r) ? (float)Gred[k * r + l] : 0.0f;
    }
  double qacc[NQ];
#pragma unroll
  for (int u = 0; u < NQ; ++u) qacc[u] = 0.0;
  const int64_t nblk = (n + UPD_B - 1) / UPD_B;
  for (int64_t blk = blockIdx.x; blk < nblk; blk += gridDim.x) {
    const int64_t j0 = blk * UPD_B;
    const int cols = (int)min((int64_t)UPD_B, n - j0);
    __syncthreads();
    for (int e = tid; e < R * UPD_B; e += UPD_THREADS) {
      const int k = e / UPD_B, c = e % UPD_B;
      Ho[k][c] = (k < r && c < cols) ? H[(int64_t)k * n + j0 + c] : 0.0f;
    }
    if (update) {
      const int len = cols * r;
      const int64_t nr = n * r;
      double acc[U];
#pragma unroll
      for (int q = 0; q < U; ++q) acc[q] = 0.0;
      for (int b = 0; b < nS; ++b) {
        const double* src = Spart + (int64_t)b * nr + j0 * r;
        double v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int e = tid + q * UPD_THREADS;
          v[q] = e < len ? __ldcg(src + e) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < U; ++q) acc[q] += v[q];
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const int e = tid + q * UPD_THREADS;
        if (e < len) Ss[(e / r) * R + e % r] = acc[q];
      }
    }
    __syncthreads();
    {
      const int c = tid >> 2, kq = tid & 3;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int k = kq + 4 * u;
        float hn = Ho[k][c];
        if (update && k < r && c < cols) {
          float e = 0.0f;
#pragma unroll
          for (int l = 0; l < R; ++l) e = fmaf(Gs[k * R + l], Ho[l][c], e);
          hn = mu_quot(hn, (float)Ss[c * R + k], e, eps);
        }
        if (k >= r || c >= cols) hn = 0.0f;
        hmax = fmaxf(hmax, hn);
        Hn[k][c] = hn;
      }
    }
    __syncthreads();
    for (int e = tid; e < R * UPD_B; e += UPD_THREADS) {
      const int k = e / UPD_B, c = e % UPD_B;
      if (c < cols) {
        const float v = Hn[k][c];
        if (update && k < r) H[(int64_t)k * n + j0 + c] = v;
        if (Hcat) {
          Hcat[(int64_t)k * ldh + j0 + c] = v;
          Hcat[(int64_t)(R + k) * ldh + j0 + c] = tf32_lo(v);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NQ; ++u) {
      const int t = tid + u * UPD_THREADS;
      if (t < rr) {
        const int k = t / r, l = t % r;
        double s0 = 0.0, s1 = 0.0;
        for (int c = 0; c < UPD_B; c += 2) {
          s0 = fma((double)Hn[k][c], (double)Hn[l][c], s0);
          s1 = fma((double)Hn[k][c + 1], (double)Hn[l][c + 1], s1);
        }
        qacc[u] += s0 + s1;
      }
    }
  }
#pragma unroll
  for (int u = 0; u < NQ; ++u) {
    const int t = tid + u * UPD_THREADS;
    if (t < rr) Qpart[(int64_t)blockIdx.x * rr + t] = qacc[u];
  }
  if (maxh) {  // max |H| for the fp16x2 scale (fp16 variant)
    for (int o = 16; o > 0; o >>= 1) hmax = fmaxf(hmax, __shfl_xor_sync(0xffffffffu, hmax, o));
    if ((tid & 31) == 0) atomicMax(maxh, __float_as_uint(hmax));
  }
}

__global__ void k_tc_sum(const double* __restrict__ part, int nparts, int len, double* __restrict__ out) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < len; t += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nparts; ++b) s += part[(int64_t)b * len + t];
    out[t] = s;
  }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 g_enc = nullptr;

cudaError_t enc() {
  if (g_enc) return cudaSuccess;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  if (e != cudaSuccess) return e;
  if (qr != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
  g_enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return cudaSuccess;
}

cudaError_t map2d(CUtensorMap* map, const float* base, uint64_t cols, uint64_t rows, uint64_t ld, uint32_t bc,
                  uint32_t br) {
  cudaError_t e = enc();
  if (e != cudaSuccess) return e;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * sizeof(float)};
  cuuint32_t box[2] = {bc, br};
  cuuint32_t es[2] = {1, 1};
  CUresult res = g_enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int rcls(int r) { return r <= 16 ? 16 : 32; }

template <int R>
int tc_stages() {
  int s = (int)((227u * 1024u - 2048u) / TcCfg<R>::SB);
  return std::min(s, 8);
}
template <int R>
size_t tc_smem(int ns) {
  return (size_t)ns * TcCfg<R>::SB + 2048;
}

// split-K choice: units = nmb * nsplit spread over `grid` persistent CTAs;
// smallest nsplit whose wave efficiency is >= 0.9 with >= 8 K tiles per unit.
void pick_split(int64_t nmb, int64_t ktiles, int grid, int* nsplit, int64_t* kchunk) {
  int best = 1;
  double beff = -1.0;
  for (int s = 1; s <= 64; ++s) {
    int64_t kc = (ktiles + s - 1) / s;
    if (s > 1 && kc < 8) break;
    int64_t ns = (ktiles + kc - 1) / kc;
    int64_t units = nmb * ns;
    int64_t waves = (units + grid - 1) / grid;
    double eff = (double)units / (double)(waves * grid);
    if (eff > beff + 1e-9) {
      beff = eff;
      best = (int)ns;
    }
    if (eff >= 0.9) break;
  }
  *nsplit = best;
  *kchunk = (ktiles + best - 1) / best;
}

template <int R, int MODE>
cudaError_t launch_skinny(const CUtensorMap& ma, const CUtensorMap& mb, int64_t Mtot, int64_t ktiles, int nsplit,
                          int64_t kchunk, int grid, int r, double* part, int evict_first, cudaStream_t st) {
  const int ns = tc_stages<R>();
  const size_t sm = tc_smem<R>(ns);
  cudaError_t e = smem_optin((const void*)(k_skinny_tc<R, MODE>), sm);
  if (e != cudaSuccess) return e;
  k_skinny_tc<R, MODE><<<grid, TC_THREADS, sm, st>>>(ma, mb, Mtot, ktiles, nsplit, kchunk, ns, 32, r, part,
                                                     evict_first);
  return cudaGetLastError();
}

}  // namespace

// ---------------------------------------------------------------- public ----
bool tc_supported(int64_t m, int64_t n, int r, int64_t ldx, const void* X) {
  if (r < 1 || r > 32) return false;
  if (m < 256 || n < 256) return false;  // short-wide unfoldings take the fused 1-pass kernels
  if ((ldx & 3) != 0) return false;
  if ((reinterpret_cast<uintptr_t>(X) & 15) != 0) return false;
  return true;
}

TcPlan plan_tc(int64_t m, int64_t n, int r, int num_sms) {
  TcPlan p;
  p.m = m;
  p.n = n;
  p.r = r;
  p.R = rcls(r);
  p.grid = num_sms;
  p.ldh = (n + 3) & ~int64_t(3);
  p.ldw = (m + 3) & ~int64_t(3);
  pick_split((m + TC_BM - 1) / TC_BM, (n + TC_BK - 1) / TC_BK, num_sms, &p.splitW, &p.kchW);
  pick_split((n + TC_BM - 1) / TC_BM, (m + TC_BK - 1) / TC_BK, num_sms, &p.splitH, &p.kchH);
  p.nG = (int)((m + UPD_B - 1) / UPD_B);
  p.nQ = (int)std::min<int64_t>((n + UPD_B - 1) / UPD_B, 4 * num_sms);  // H-update CTAs (grid-stride)
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t at = o;
    o = (o + b + 255) & ~size_t(255);
    return at;
  };
  p.off_hcat = take(sizeof(float) * (size_t)(2 * p.R) * p.ldh);
  p.off_wcat = take(sizeof(float) * (size_t)(2 * p.R) * p.ldw);
  p.off_P = take(sizeof(double) * (size_t)p.splitW * m * r);
  p.off_S = take(sizeof(double) * (size_t)p.splitH * n * r);
  p.off_G = take(sizeof(double) * (size_t)p.nG * r * r);
  p.off_Q = take(sizeof(double) * (size_t)p.nQ * r * r);
  p.off_Gred = take(sizeof(double) * (size_t)r * r);
  p.off_Qred = take(sizeof(double) * (size_t)r * r);
  p.off_red = take(sizeof(double) * (size_t)(m * r + r * r));  // distributed: [P | Q] all-reduce payload
  p.off_Sred = take(sizeof(double) * (size_t)n * r);          // distributed: W^T X block payload
  // fp16x2 variant (mu_tc16.cu): default unless NTT_TC16=0
  {
    const char* e = getenv("NTT_TC16");
    p.f16 = !(e && e[0] == '0');
  }
  p.ldh16 = (n + 7) & ~int64_t(7);
  p.ldw16 = (m + 7) & ~int64_t(7);
  pick_split((m + TC_BM - 1) / TC_BM, (n + 63) / 64, num_sms, &p.splitW16, &p.kchW16);
  pick_split((n + TC_BM - 1) / TC_BM, (m + 63) / 64, num_sms, &p.splitH16, &p.kchH16);
  if (p.f16) {  // the split partial buffers must hold either variant's split count
    p.off_P = take(sizeof(double) * (size_t)std::max(p.splitW, p.splitW16) * m * r);
    p.off_S = take(sizeof(double) * (size_t)std::max(p.splitH, p.splitH16) * n * r);
  }
  p.off_h16 = take(2 * sizeof(uint16_t) * (size_t)(2 * p.R) * p.ldh16);
  p.off_w16 = take(2 * sizeof(uint16_t) * (size_t)(2 * p.R) * p.ldw16);
  p.off_scales = take(256);
  p.bytes = o;
  return p;
}

cudaError_t tc_prepare(const TcPlan& p, const float* X, int64_t ldx, float* H, char* ws, TcMaps* maps,
                       cudaStream_t st) {
  float* Hcat = reinterpret_cast<float*>(ws + p.off_hcat);
  float* Wcat = reinterpret_cast<float*>(ws + p.off_wcat);
  cudaError_t e;
  const uint32_t N1 = 2u * (uint32_t)p.R;
  if ((e = map2d(&maps->xw, X, p.n, p.m, ldx, 32, TC_BM))) return e;
  if ((e = map2d(&maps->xh, X, p.n, p.m, ldx, 32, 32))) return e;
  if ((e = map2d(&maps->hcat, Hcat, p.n, N1, p.ldh, 32, N1))) return e;
  if ((e = map2d(&maps->wcat, Wcat, p.m, N1, p.ldw, 32, N1))) return e;
  // zero the padded rank rows once (never written afterwards)
  if ((e = cudaMemsetAsync(Hcat, 0, sizeof(float) * (size_t)N1 * p.ldh, st))) return e;
  if ((e = cudaMemsetAsync(Wcat, 0, sizeof(float) * (size_t)N1 * p.ldw, st))) return e;
  double* Qpart = reinterpret_cast<double*>(ws + p.off_Q);
  const unsigned g = (unsigned)p.nQ;
  if (p.R == 16)
    k_tc_hupdate<16><<<g, UPD_THREADS, 0, st>>>(H, p.n, p.r, nullptr, 0, nullptr, 0.f, false, Hcat, p.ldh, Qpart,
                                             nullptr);
  else
    k_tc_hupdate<32><<<g, UPD_THREADS, 0, st>>>(H, p.n, p.r, nullptr, 0, nullptr, 0.f, false, Hcat, p.ldh, Qpart,
                                             nullptr);
  return cudaGetLastError();
}

cudaError_t tc_sum_Q(const TcPlan& p, char* ws, cudaStream_t st) {
  // r^2 entries over nQ (up to 4 x 148) partials: one warp per entry (launch_sum_partials), not
  // one thread walking every partial (88 us on config 5)
  return launch_sum_partials(reinterpret_cast<double*>(ws + p.off_Q), p.nQ, (int64_t)p.r * p.r,
                             reinterpret_cast<double*>(ws + p.off_Qred), st);
}

cudaError_t tc_pass_w(const TcPlan& p, const TcMaps& mp, char* ws, int evict_first, cudaStream_t st) {
  double* P = reinterpret_cast<double*>(ws + p.off_P);
  const int64_t kt = (p.n + TC_BK - 1) / TC_BK;
  if (p.R == 16) return launch_skinny<16, 0>(mp.xw, mp.hcat, p.m, kt, p.splitW, p.kchW, p.grid, p.r, P, evict_first, st);
  return launch_skinny<32, 0>(mp.xw, mp.hcat, p.m, kt, p.splitW, p.kchW, p.grid, p.r, P, evict_first, st);
}

cudaError_t tc_wupdate(const TcPlan& p, float* W, float eps, char* ws, cudaStream_t st, int it) {
  return tc_wupdate_ex(p, W, eps, ws, reinterpret_cast<const double*>(ws + p.off_P), p.f16 ? p.splitW16 : p.splitW,
                       reinterpret_cast<const double*>(ws + p.off_Qred), st, it);
}

// fp16 variant max words (unsigned, after the 64-byte scale block): [0] X, [1 + (it & 1)] H, [3 + (it & 1)] W
static unsigned* tc_maxw(const TcPlan& p, char* ws, int slot) {
  return p.f16 ? reinterpret_cast<unsigned*>(ws + p.off_scales + 64) + slot : nullptr;
}

cudaError_t tc_wupdate_ex(const TcPlan& p, float* W, float eps, char* ws, const double* P, int nP, const double* Qr,
                          cudaStream_t st, int it) {
  float* Wcat = p.f16 ? nullptr : reinterpret_cast<float*>(ws + p.off_wcat);
  unsigned* mxw = tc_maxw(p, ws, 3 + (it & 1));
  double* G = reinterpret_cast<double*>(ws + p.off_G);
  const unsigned g = (unsigned)p.nG;
  if (p.R == 16)
    k_tc_wupdate<16><<<g, UPD_THREADS, 0, st>>>(W, p.m, p.r, P, nP, Qr, eps, Wcat, p.ldw, G, mxw);
  else
    k_tc_wupdate<32><<<g, UPD_THREADS, 0, st>>>(W, p.m, p.r, P, nP, Qr, eps, Wcat, p.ldw, G, mxw);
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  return launch_sum_partials(G, p.nG, (int64_t)p.r * p.r, reinterpret_cast<double*>(ws + p.off_Gred), st);
}

cudaError_t tc_pass_h(const TcPlan& p, const TcMaps& mp, char* ws, int evict_first, cudaStream_t st) {
  double* S = reinterpret_cast<double*>(ws + p.off_S);
  const int64_t kt = (p.m + TC_BK - 1) / TC_BK;
  if (p.R == 16) return launch_skinny<16, 1>(mp.xh, mp.wcat, p.n, kt, p.splitH, p.kchH, p.grid, p.r, S, evict_first, st);
  return launch_skinny<32, 1>(mp.xh, mp.wcat, p.n, kt, p.splitH, p.kchH, p.grid, p.r, S, evict_first, st);
}

cudaError_t tc_hupdate(const TcPlan& p, float* H, float eps, char* ws, cudaStream_t st, int it) {
  return tc_hupdate_ex(p, H, eps, ws, reinterpret_cast<const double*>(ws + p.off_S), p.f16 ? p.splitH16 : p.splitH, st,
                       it);
}

cudaError_t tc_hupdate_ex(const TcPlan& p, float* H, float eps, char* ws, const double* S, int nS, cudaStream_t st,
                          int it) {
  unsigned* mxh = tc_maxw(p, ws, 1 + (it & 1));
  const double* Gr = reinterpret_cast<const double*>(ws + p.off_Gred);
  float* Hcat = p.f16 ? nullptr : reinterpret_cast<float*>(ws + p.off_hcat);
  double* Q = reinterpret_cast<double*>(ws + p.off_Q);
  const unsigned g = (unsigned)p.nQ;
  if (p.R == 16)
    k_tc_hupdate<16><<<g, UPD_THREADS, 0, st>>>(H, p.n, p.r, S, nS, Gr, eps, true, Hcat, p.ldh, Q, mxh);
  else
    k_tc_hupdate<32><<<g, UPD_THREADS, 0, st>>>(H, p.n, p.r, S, nS, Gr, eps, true, Hcat, p.ldh, Q, mxh);
  return cudaGetLastError();
}

// distributed: red = [sum of the P split partials | Q]  (payload of the grid-row all-reduce)
cudaError_t tc_reduce_PQ(const TcPlan& p, char* ws, cudaStream_t st) {
  double* red = reinterpret_cast<double*>(ws + p.off_red);
  const int64_t mr = p.m * p.r;
  k_tc_sum<<<(unsigned)std::min<int64_t>((mr + 255) / 256, 1184), 256, 0, st>>>(
      reinterpret_cast<const double*>(ws + p.off_P), p.f16 ? p.splitW16 : p.splitW, (int)mr, red);
  cudaError_t e = cudaGetLastError();
  if (e) return e;
  return cudaMemcpyAsync(red + mr, ws + p.off_Qred, sizeof(double) * p.r * p.r, cudaMemcpyDeviceToDevice, st);
}

// distributed: Sred = sum of the S split partials (payload of the grid-column all-reduce)
cudaError_t tc_reduce_S(const TcPlan& p, char* ws, cudaStream_t st) {
  const int64_t nr = p.n * p.r;
  k_tc_sum<<<(unsigned)std::min<int64_t>((nr + 255) / 256, 1184), 256, 0, st>>>(
      reinterpret_cast<const double*>(ws + p.off_S), p.f16 ? p.splitH16 : p.splitH, (int)nr,
      reinterpret_cast<double*>(ws + p.off_Sred));
  return cudaGetLastError();
}

}  // namespace ntt
