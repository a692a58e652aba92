// mu_fused.cu -- the 1-pass fused MU kernel for short-wide unfoldings (m <= 40,
// r <= 8) on sm_100a, plus the parallel-reduction W update it feeds.
//
// One pass over X does, per column j (include/ntt.h ntt_nmf_mu; R1-R4):
//   phase A  S[:,j] = W^T X[:,j]                          (Alg. 6 l.2)
//            H[:,j] <- H[:,j] o S[:,j] / (G H[:,j] + eps)  (G = W^T W, Alg. 4)
//   phase B  P += X[:,j] Hn[:,j]^T,  Q += Hn[:,j] Hn[:,j]^T (Alg. 5 l.2 / Alg. 4
//            for the NEXT iteration's W update)
// so X is read from HBM once per MU iteration instead of twice (SURVEY s.0 #3).
//
// Structure: persistent CTAs (1 per SM), 1 TMA producer warp + 8 consumer warps.
// The producer streams tiles of 128 columns -- X as four 32-column x MP-row
// boxes and H as four 32 x 8 boxes, all SWIZZLE_128B -- through an mbarrier
// ring of `ns` stages.  Each consumer warp owns whole tiles (no CTA-wide syncs
// in the loop): lane q handles columns 4q..4q+3 in phase A (FFMA2 with scalar
// broadcast of W), then the warp re-reads its tile for phase B with lanes as
// (row block rb, 32-column slice cs) -- rows rb+8u hit distinct swizzle phases,
// so the 128-bit loads are conflict-free -- against a transposed, padded Hn tile
// read by broadcast.  fp32 FMA inside a tile, fp64 accumulation across tiles,
// fixed-order CTA reduction into per-CTA fp64 partials (deterministic).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <utility>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "mu_fused.h"
#include "sm100.cuh"

namespace ntt {

namespace {

constexpr int NW = 8;               // consumer warps
constexpr int NT = (NW + 1) * 32;   // + 1 TMA producer warp
constexpr int BN = 128;             // tile columns
constexpr int HN_FLOATS = 1168;     // per-warp transposed Hn tile (padded)
constexpr int SMEM_BUDGET = 232448; // 227 KB opt-in

using namespace sm100;  // mbarrier / TMA wrappers (sm100.cuh)

#ifdef NTT_WATCHDOG
__device__ __forceinline__ void mbar_wait_dbg(uint64_t* bar, uint32_t parity, int tag, long long j) {
  long long t0 = clock64();
  while (true) {
    if (mbar_try(bar, parity)) return;
    if (clock64() - t0 > 4000000000LL) {
      printf("WATCHDOG tag=%d block=%d thread=%d j=%lld parity=%u\n", tag, blockIdx.x, threadIdx.x, j, parity);
      __trap();
    }
  }
}
#define MBAR_WAIT(bar, par, tag, j) mbar_wait_dbg(bar, par, tag, j)
#else
#define MBAR_WAIT(bar, par, tag, j) mbar_wait(bar, par)
#endif
#ifdef NTT_WATCHDOG
#define MBAR_WAIT_BACKOFF(bar, par, tag, j) mbar_wait_dbg(bar, par, tag, j)
#else
// producer-side wait with a sleep between polls: a spinning producer warp takes issue
// slots from the consumer warp sharing its scheduler (k_fused_c: 24 % of all executed
// instructions were this poll, ncu source page)
#define MBAR_WAIT_BACKOFF(bar, par, tag, j) \
  do {                                     \
    while (!mbar_try_sleep(bar, par)) {     \
    }                                      \
  } while (0)
#endif
__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ float4 lds128(const unsigned char* p) {
  return *reinterpret_cast<const float4*>(p);
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
// MU quotient (w * num) / (den + eps) (reading R4) with the 2-ulp fast divide
__device__ __forceinline__ float mu_q(float w, float num, float den, float eps) {
  return __fdividef(__fmul_rn(w, num), __fadd_rn(den, eps));
}
__device__ __forceinline__ float2 bc(float a) { return make_float2(a, a); }

// transposed per-warp Hn tile: column c (0..127), rank index k (0..7)
__device__ __forceinline__ int hn_idx(int c, int k) { return c * 8 + k + 4 * (c >> 2) + 4 * (c >> 5); }
// transposed Hn tile stored over the stage's (already consumed) H boxes: 8 floats
// per column, row rho(c) = c ^ (((c >> 2) + c / SL) & 3) -- conflict-free phase-B
// reads (the 4 column slices land in distinct bank groups), 2-way phase-A writes.
template <int SL>
__device__ __forceinline__ int hn_sw(int c, int k) { return ((c ^ (((c >> 2) + c / SL) & 3)) << 3) + k; }

// ---------------------------------------------------------------------------
// Persistent mode (PersistArgs.iters > 0): ONE cooperative launch runs the whole
// MU loop of a TT step -- the acc-only prologue pass (P0 = X H0^T, Q0 = H0 H0^T)
// and `iters` fused passes.  Between passes every CTA writes its fp64 (P, Q)
// partial ([P (m r) | Q (r r)], L doubles) to part[cta], then
//   grid barrier -> CTA b sums slice b of the L entries over all CTAs (fixed
//   order) into red -> grid barrier -> every CTA computes the SAME W update
//   W <- W o P / (W Q + eps) (fp64, reading R4) and G = W^T W in its own smem.
// This replaces the per-iteration W-update launch and the pass launch (~20 us of
// launch/ramp/partial traffic per iteration on small TT steps).
// ---------------------------------------------------------------------------

__device__ __forceinline__ void pstamp(const PersistArgs& pa, int it, int ph) {
  if (pa.trace && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (blockIdx.x == 0) pa.trace[it * 4 + ph] = t;
    // per-CTA end of pass 1 (load-balance diagnostics): [16384 + cta], start of pass 1: [17408 + cta]
    if (it == 1 && ph == 1 && blockIdx.x < 1024) pa.trace[16384 + blockIdx.x] = t;
    if (it == 1 && ph == 0 && blockIdx.x < 1024) pa.trace[17408 + blockIdx.x] = t;
    // passes 2..4: per-CTA ends at [18432 + 1024 (it - 2) + cta]; the CTA's SM at [21504 + cta]
    if (it >= 2 && it <= 4 && ph == 1 && blockIdx.x < 1024) pa.trace[18432 + 1024 * (it - 2) + blockIdx.x] = t;
    if (it == 1 && ph == 0 && blockIdx.x < 1024) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      pa.trace[21504 + blockIdx.x] = smid;
    }
  }
}

// fine-grained diagnostics inside persist_step: [12288 + 4 it + k], k < 4, CTA 0 only
__device__ __forceinline__ void pstamp2(const PersistArgs& pa, int it, int k) {
  if (pa.trace && threadIdx.x == 0 && blockIdx.x == 0 && it < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    pa.trace[12288 + it * 4 + k] = t;
    pa.trace[8192 + it * 4 + k] = (unsigned long long)clock64();
  }
}

__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// grid-wide barrier over co-resident CTAs (cooperative launch).  The proxy fence
// orders this thread's generic global writes (H) before later TMA (async-proxy)
// reads of the same data by any CTA.
__device__ __forceinline__ void grid_sync(unsigned* ctr, unsigned& epoch) {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  epoch += gridDim.x;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (ld_acquire_gpu(ctr) < epoch) {
    }
    __threadfence();
  }
  __syncthreads();
}

// ---- cross-GPU exchange (PersistArgs::xpeers; SURVEY s.8(e)): system-scope flags
__device__ __forceinline__ unsigned long long* xflags(double* base, int nranks) {
  return reinterpret_cast<unsigned long long*>(base + 2 * (size_t)nranks * kXLmax);
}
__device__ __forceinline__ unsigned long long xseq_load(const PersistArgs& pa) {
  if (pa.nranks <= 0) return 0ull;
  const unsigned long long* sp = xflags(pa.xpeers[pa.rank], pa.nranks) + 2 * pa.nranks;
  return *reinterpret_cast<const volatile unsigned long long*>(sp);
}
// end of a persistent launch: advance the buffer's pass counter (CTA 0, after the last barrier)
__device__ __forceinline__ void xseq_store(const PersistArgs& pa, unsigned long long xs0) {
  if (pa.nranks > 0 && blockIdx.x == 0 && threadIdx.x == 0)
    *(xflags(pa.xpeers[pa.rank], pa.nranks) + 2 * pa.nranks) = xs0 + (unsigned long long)pa.iters;
}
__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// CTA 0: stage this GPU's reduced vector src (L doubles, L2) in shared memory (one round trip:
// all 8 loads of a thread issued together), store it into slot [par][rank] of every rank's
// buffer, then one thread per rank: fence + release flag [par][rank] on that rank.
__device__ void xpush(const PersistArgs& pa, const double* src, int L, unsigned long long seq, double* stg) {
  const int p = pa.nranks, T = blockDim.x, tid = threadIdx.x;
  const int par = (int)(seq & 1ull);
  for (int e0 = 0; e0 < L; e0 += 8 * T) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q * T + tid;
      v[q] = e < L ? __ldcg(src + e) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q * T + tid;
      if (e < L) stg[e] = v[q];
    }
  }
  __syncthreads();
  for (int q = 0; q < p; ++q) {
    double* dst = pa.xpeers[q] + ((size_t)par * p + pa.rank) * kXLmax;
    for (int e = tid; e < L; e += T) dst[e] = stg[e];
  }
  __syncthreads();
  if (tid < p) {
    __threadfence_system();
    st_release_sys_u64(xflags(pa.xpeers[tid], p) + par * p + pa.rank, seq);
  }
}

// every CTA: wait until all ranks' flags [par][*] of the own buffer carry seq (acquire, system
// scope), so the slot reads that follow see the peers' stores
__device__ void xwait(const PersistArgs& pa, unsigned long long seq) {
  const int p = pa.nranks, tid = threadIdx.x;
  if (tid < p) {
    const unsigned long long* f = xflags(pa.xpeers[pa.rank], p) + (int)(seq & 1ull) * p + tid;
    while (ld_acquire_sys_u64(f) < seq) {
    }
  }
  __syncthreads();
}

// Reduce the per-CTA partials and apply the W update in every CTA (see above).
// Scratch layout (doubles): P (m r) | Qp (RK x RK, Q zero-padded) | Wd (m RK, W as fp64) |
// Wnd (m RK, new W rounded to fp32, held as fp64) | Gp ([<= T / RK chunks][RK][RK] Gram partials).
// RK = 8 or 16 (the kernel's padded rank); Ws / Wnd layout [i RK + k], ranks >= r stay 0.
__host__ __device__ constexpr int64_t persist_scratch_doubles(int64_t m, int r, int rk, int threads) {
  return m * r + 1 + (int64_t)rk * rk + 2 * m * rk + (int64_t)(threads / rk) * rk * rk;
}

template <int RK>
__device__ void persist_step(const PersistArgs& pa, unsigned& epoch, int m, int r, float eps, float* Ws, float* Gs,
                             double* scr, int it, unsigned long long xs0) {
  const int L = m * r + r * r;
  const int T = blockDim.x, tid = threadIdx.x;
  pstamp(pa, it, 1);
  if (gridDim.x > 1) {
    grid_sync(pa.ctr, epoch);
    pstamp(pa, it, 2);
    const int G = gridDim.x;
    const int NP = G + 8 * pa.tail_groups;  // partial slots: one per CTA, then the dynamic tail's
    const int SL = (L + G - 1) / G;
    const int e0 = blockIdx.x * SL;
    const int ne = min(L, e0 + SL) - e0;
    if (ne > 0) {
      // slice [e0, e0 + ne) summed over the NP partials: (entry, chunk of partials) per thread, all
      // loads of a chunk (<= 16) issued before any is used (one L2 round trip)
      int C = T / ne;
      C = C < 1 ? 1 : (C > 96 ? 96 : C);
      for (int t = tid; t < ne * C; t += T) {
        const int e = t % ne, c = t / ne;
        const int g0 = (int)((int64_t)NP * c / C), g1 = (int)((int64_t)NP * (c + 1) / C);
        const double* src = pa.part + e0 + e;
        double acc = 0.0;
        for (int gb = g0; gb < g1; gb += 16) {
          double a[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) a[q] = (gb + q < g1) ? __ldcg(src + (int64_t)(gb + q) * L) : 0.0;
          acc += (((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]))) +
                 (((a[8] + a[9]) + (a[10] + a[11])) + ((a[12] + a[13]) + (a[14] + a[15])));
        }
        scr[c * ne + e] = acc;
      }
      __syncthreads();
      // the C chunk sums of an entry: a warp per entry, lane l adds chunks l, l + 32, ... in order,
      // then a fixed xor butterfly (a sequential loop over C <= 96 chunks was ~1.5 us)
      const int wid = tid >> 5, ln = tid & 31;
      for (int e = wid; e < ne; e += (T >> 5)) {
        double sv = 0.0;
        for (int c = ln; c < C; c += 32) sv += scr[c * ne + e];
        sv = warp_sum(sv);
        if (ln == 0) __stcg(pa.red + e0 + e, sv);
      }
    }
    grid_sync(pa.ctr, epoch);
  } else {
    __syncthreads();  // single CTA: its own partial is the sum
  }
  const double* srcv = gridDim.x > 1 ? pa.red : pa.part;
  const unsigned long long seq = xs0 + (unsigned long long)it + 1ull;
  if (pa.nranks > 0) {  // every rank's vector into every rank's slots (see PersistArgs::xpeers)
    if (blockIdx.x == 0) xpush(pa, srcv, L, seq, scr);
    xwait(pa, seq);
  }
  pstamp(pa, it, 3);
  double* P = scr;                 // m x r
  double* Qp = scr + ((m * r + 1) & ~1);  // RK x RK (16-byte aligned for the double2 loads)
  double* Wd = Qp + RK * RK;       // m x RK
  double* Wnd = Wd + m * RK;       // m x RK
  double* Gp = Wnd + m * RK;       // [GC][RK][RK]
  // (P, Q) into shared memory: coalesced, all 16 loads of a thread issued before any is used
  // (one L2 round trip for L <= 16 T: m = 256, r = 8 at 160 threads)
  const double* xslots = pa.nranks > 0 ? pa.xpeers[pa.rank] + (size_t)(seq & 1ull) * pa.nranks * kXLmax : nullptr;
  constexpr int NV = 16;
  for (int e0 = 0; e0 < L; e0 += NV * T) {
    double v[NV];
    if (pa.nranks > 0) {  // sum of the ranks' vectors in rank order (identical on every rank)
#pragma unroll
      for (int q = 0; q < NV; ++q) v[q] = 0.0;
#pragma unroll 4
      for (int sr = 0; sr < pa.nranks; ++sr) {
        const double* sl = xslots + (size_t)sr * kXLmax;
#pragma unroll
        for (int q = 0; q < NV; ++q) {
          const int e = e0 + q * T + tid;
          if (e < L) v[q] += __ldcg(sl + e);
        }
      }
    } else {
#pragma unroll
      for (int q = 0; q < NV; ++q) {
        const int e = e0 + q * T + tid;
        v[q] = e < L ? __ldcg(srcv + e) : 0.0;
      }
    }
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int e = e0 + q * T + tid;
      if (e < m * r) P[e] = v[q];
      else if (e < L) {
        const int f = e - m * r;
        Qp[(f / r) * RK + f % r] = v[q];
      }
    }
  }
  for (int e = tid; e < RK * RK; e += T)
    if ((e / RK) >= r || (e % RK) >= r) Qp[e] = 0.0;
  for (int e = tid; e < m * RK; e += T) Wd[e] = (double)Ws[e];
  __syncthreads();
  pstamp2(pa, it, 0);
  // W <- W o P / (W Q + eps) (fp64, reading R4): thread (rank kq = tid % RK, row group) keeps
  // column kq of Q in registers and walks rows tid / RK, + T / RK, ...: one quotient per row and
  // thread (independent across the unrolled rows; a thread owning whole rows serialised RK
  // quotients), the d = sum_l W[i][l] Q[l][kq] chain in the same order as before
  {
    const int kq = tid % RK, di = T / RK;
    double qc[RK];
#pragma unroll
    for (int l = 0; l < RK; ++l) qc[l] = Qp[l * RK + kq];
#pragma unroll 2
    for (int i = tid / RK; i < m; i += di) {
      double w[RK];
#pragma unroll
      for (int l = 0; l < RK; l += 2) {
        const double2 v = *reinterpret_cast<const double2*>(Wd + i * RK + l);
        w[l] = v.x;
        w[l + 1] = v.y;
      }
      double d = 0.0;
#pragma unroll
      for (int l = 0; l < RK; ++l) d = fma(w[l], qc[l], d);
      const double wk = Wd[i * RK + kq];  // not w[kq]: a run-time index puts w in local memory
      Wnd[i * RK + kq] = kq < r ? (double)(float)mu_quot_fast(wk, P[i * r + kq], d, (double)eps) : 0.0;
    }
  }
  __syncthreads();
  pstamp2(pa, it, 1);
#pragma unroll 4
  for (int e = tid; e < m * RK; e += T) Ws[e] = (float)Wnd[e];
  // G = Wn^T Wn: thread (k, chunk c) accumulates row k of G over the chunk's rows (RK
  // independent chains); chunks summed in fixed order below
  const int GC = T / RK;
  for (int t = tid; t < RK * GC; t += T) {
    const int k = t % RK, c = t / RK;
    const int i0 = m * c / GC, i1 = m * (c + 1) / GC;  // m <= 256: 32-bit
    double g[RK];
#pragma unroll
    for (int l = 0; l < RK; ++l) g[l] = 0.0;
#pragma unroll 4
    for (int i = i0; i < i1; ++i) {
      const double wk = Wnd[i * RK + k];
#pragma unroll
      for (int l = 0; l < RK; l += 2) {
        const double2 v = *reinterpret_cast<const double2*>(Wnd + i * RK + l);
        g[l] = fma(wk, v.x, g[l]);
        g[l + 1] = fma(wk, v.y, g[l + 1]);
      }
    }
#pragma unroll
    for (int l = 0; l < RK; ++l) Gp[(c * RK + k) * RK + l] = g[l];
  }
  __syncthreads();
  pstamp2(pa, it, 2);
  for (int e = tid; e < RK * RK; e += T) {
    double sg = 0.0;
#pragma unroll 4
    for (int c = 0; c < GC; ++c) sg += Gp[c * RK * RK + e];
    Gs[e] = ((e / RK) < r && (e % RK) < r) ? (float)sg : 0.0f;
  }
  if (blockIdx.x == 0 && it == pa.iters - 1)  // the final W (later passes only update H)
    for (int e = tid; e < m * r; e += T) pa.Wout[e] = (float)Wnd[(e / r) * RK + (e % r)];
  __syncthreads();
  pstamp2(pa, it, 3);
}

template <int R, int UX, int NWT, bool HDIRECT, int BNT, bool FOLD>
__global__ void __launch_bounds__((NWT + 1) * 32, 1)
k_fused(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmH,
        const __grid_constant__ CUtensorMap tmH2, int m, int64_t n, int r,
        const float* __restrict__ W, const double* __restrict__ Gpart, int nG, float eps, float* __restrict__ H,
        double* __restrict__ Ppart, double* __restrict__ Qpart, int mode, int ns, int evict_first,
        PersistArgs pa) {
  extern __shared__ unsigned char smem_raw[];
  // keep the shared address space visible to the compiler (LDS/STS, not generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int MP = UX * 8;                 // padded rows (TMA box rows)
  constexpr int NB = BNT / 32;               // 32-column boxes per tile
  constexpr int CPL = BNT / 32;              // phase-A columns per lane (4 or 2)
  constexpr int SL = BNT / 4;                // phase-B columns per slice lane-group
  constexpr uint32_t XB = (uint32_t)NB * MP * 128u;
  // Small m (UX <= 2): H is NOT staged -- lanes read their H columns with
  // coalesced 128-bit global loads issued before the stage wait, so stages are
  // small and many are in flight (H is most of the traffic there).  Larger m:
  // H rides in the stage as four 32 x 8 TMA boxes.
  constexpr uint32_t HB = HDIRECT ? 0u : (uint32_t)NB * 8u * 128u;
  // FOLD (BCD one-pass, PersistArgs::bcdFold): a second set of H boxes per stage, B[role]
  static_assert(!(FOLD && HDIRECT), "k_fused: the H_m fold needs staged H");
  constexpr uint32_t SB = XB + HB * (FOLD ? 2u : 1u);
  unsigned char* stages = smem;
  float* Ws = reinterpret_cast<float*>(smem + (size_t)ns * SB);  // MP x 8
  float* Gs = Ws + MP * 8;                                         // 8 x 8
  // HDIRECT: per-warp padded Hn tiles; otherwise Hn overwrites the stage's H boxes
  float* HnAll = Gs + 64;                                          // NWT x HN_FLOATS (HDIRECT)
  uint64_t* full = reinterpret_cast<uint64_t*>(HnAll + (HDIRECT ? NWT * HN_FLOATS : 0));
  uint64_t* empty = full + ns;
  // Dynamic stage assignment (no head-of-line blocking between the warp-owned
  // tiles): the producer loads tile `pos` into ANY free stage s (bit s of
  // free_mask, set again by the consuming warp when it is done), tags the stage
  // tag[s] = pos << 1 | fill parity and then publishes issued = pos + 1
  // (release).  The consumer, after acquiring `issued`, finds the stage whose tag
  // holds its pos (one ballot over the <= 24 tags).  A stage's tag cannot change
  // before its consumer releases it, so there is no overrun however far the
  // other warps run ahead (a 32-entry pos % 32 slot ring could be overwritten).
  uint32_t* issued = reinterpret_cast<uint32_t*>(empty + ns);
  uint32_t* free_mask = issued + 1;
  uint32_t* tag = issued + 2;  // [ns <= 24]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool persist = pa.iters > 0;
  // FOLD: H_m = diag(a) B[1 - role] - diag(b) B[role] (B = tmH, tmH2 over Hout, Hout2); the
  // second box set is loaded only when some b_k != 0 (after an accepted iteration)
  const bool role1 = FOLD && *pa.bcdRole != 0.0;
  bool ext = false;
  if (FOLD)
    for (int l = 0; l < r; ++l) ext |= pa.bcdS[64 + l] != 0.0;

  // ---- setup: W, G into smem; barriers
  for (int e = tid; e < MP * 8; e += (NWT + 1) * 32) {
    int i = e >> 3, k = e & 7;
    Ws[e] = (i < m && k < r) ? W[(int64_t)i * r + k] : 0.0f;
  }
  if (!persist && (mode & kFusedUpdate)) {
    const int rr = r * r;
    for (int e = tid; e < 64; e += (NWT + 1) * 32) {
      int k = e >> 3, l = e & 7;
      double s = 0.0;
      if (k < r && l < r)
        for (int b = 0; b < nG; ++b) s += Gpart[(int64_t)b * rr + k * r + l];
      Gs[e] = (float)s;
    }
  }
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    *issued = 0u;
    *free_mask = (ns >= 32) ? 0xffffffffu : ((1u << ns) - 1u);
    for (int q = 0; q < ns; ++q) tag[q] = 0xffffffffu;  // never a valid pos << 1 | parity
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t par_mask = 0u;  // producer: parity of the next fill of each stage

  const int64_t ntiles = (n + BNT - 1) / BNT;
  const int64_t b = blockIdx.x;
  const int64_t J = (ntiles > b) ? (ntiles - b + gridDim.x - 1) / gridDim.x : 0;

  unsigned epoch = 0;
  const int nit = persist ? pa.iters + 1 : 1;
  const unsigned long long xs0 = persist ? xseq_load(pa) : 0ull;
  for (int it = 0; it < nit; ++it) {
  // persistent: pass 0 = acc-only prologue, passes 1..iters update (+ acc except the last)
  const int md = persist ? (it == 0 ? kFusedAcc : (kFusedUpdate | (it < pa.iters ? kFusedAcc : 0))) : mode;
  const bool do_update = (md & kFusedUpdate) != 0;
  const bool do_acc = (md & kFusedAcc) != 0;
  const int64_t pbase = (int64_t)it * J;  // ring position of this pass's first tile
  pstamp(pa, it, 0);
  if (warp == NWT) {
    // ================= TMA producer =================
    if (lane == 0) {
      uint64_t policy;
      if (evict_first & 1)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
      const bool x3d = (evict_first & 2) != 0;  // tmX is the 3-D map: the tile's NB boxes in one transaction
      for (int64_t j = 0; j < J; ++j) {
        const int64_t pos = pbase + j;
        uint32_t fm;
        while ((fm = ld_acquire_u32(free_mask)) == 0u) {
        }
        const int s = __ffs(fm) - 1;
        atomicAnd(free_mask, ~(1u << s));
        const uint32_t ph = (par_mask >> s) & 1u;
        par_mask ^= 1u << s;
        tag[s] = ((uint32_t)pos << 1) | ph;
        mbar_expect_tx(&full[s], XB + (HDIRECT ? 0u : HB) + (FOLD && ext ? HB : 0u));
        const int col0 = (int)((b + j * gridDim.x) * BNT);
        unsigned char* st = stages + (size_t)s * SB;
        if (x3d) {
          tma_load_3d(st, &tmX, 0, 0, col0 >> 5, &full[s], policy);
        } else {
#pragma unroll
          for (int bx = 0; bx < NB; ++bx) tma_load_2d(st + bx * MP * 128, &tmX, col0 + bx * 32, 0, &full[s], policy);
        }
        if (!HDIRECT) {
          // FOLD: H_prev = B[1 - role] into the usual boxes, B[role] (H_prev2) after them
          const CUtensorMap* mp = (FOLD && !role1) ? &tmH2 : &tmH;
          const CUtensorMap* mq = role1 ? &tmH2 : &tmH;
          if (x3d) {
            tma_load_3d(st + XB, mp, 0, 0, col0 >> 5, &full[s], policy);
            if (FOLD && ext) tma_load_3d(st + XB + HB, mq, 0, 0, col0 >> 5, &full[s], policy);
          } else {
#pragma unroll
            for (int bx = 0; bx < NB; ++bx) tma_load_2d(st + XB + bx * 1024, mp, col0 + bx * 32, 0, &full[s], policy);
            if (FOLD && ext)
#pragma unroll
              for (int bx = 0; bx < NB; ++bx)
                tma_load_2d(st + XB + HB + bx * 1024, mq, col0 + bx * 32, 0, &full[s], policy);
          }
        }
        st_release_u32(issued, (uint32_t)(pos + 1));
      }
    }
  } else {

  // ================= consumer warps =================
  float* HwDirect = HnAll + warp * HN_FLOATS;
  // phase A: lane q owns columns cq..cq+CPL-1 (box qbox, 16B chunk qch, float offset qsub)
  const int q = lane, cq = q * CPL, qbox = cq >> 5, qch = (cq & 31) >> 2, qsub = cq & 3;
  const int rb = lane & 7, cs = lane >> 3;  // phase B: rows rb+8u, columns cs*SL .. cs*SL+SL-1
  // phase-B accumulators: V4 = (UX+1)*R values per lane (rows rb+8u, u<UX, and Q
  // row rb), padded to a multiple of 4.  After every tile the 4 lanes sharing rb
  // (cs = 0..3) reduce-scatter them with two shuffle levels, so each lane keeps
  // V4/4 of the sums, flat indices [cs*V4/4, cs*V4/4 + V4/4), in fp64.
  constexpr int V = (UX + 1) * R;
  constexpr int V4 = (V + 3) / 4 * 4;
  double accd[V4 / 4];
#pragma unroll
  for (int v = 0; v < V4 / 4; ++v) accd[v] = 0.0;
  const bool h1 = (lane >> 4) & 1, h0 = (lane >> 3) & 1;
  // phase-B fp32 accumulators live across RS tiles; the reduce-scatter + fp64 fold
  // runs every RS tiles (and after the warp's last tile): <= RS * SL / 4 fp32 terms
  constexpr int RS = 1;  // reduce-scatter every tile (4 measured within noise, more registers)
  float2 acc[V4 / 2];
#pragma unroll
  for (int v = 0; v < V4 / 2; ++v) acc[v] = f2(0.f, 0.f);
  int ntile = 0;
  // swizzle offsets: phase A row i reads chunk (qch ^ (i & 7)), phase B chunk (s4 ^ rb)

  // HDIRECT: this lane's H columns of a tile, loaded ONE TILE AHEAD (software
  // pipelined: the global-load latency overlaps the previous tile's work; each
  // tile's H is only read and written by its owning warp, so the early read is safe)
  auto load_h = [&](int64_t jj, float2 (&dst)[R][CPL / 2]) {
    const int64_t cc = (b + jj * gridDim.x) * BNT + cq;
#pragma unroll
    for (int l = 0; l < R; ++l) {
      float hx[4] = {0.f, 0.f, 0.f, 0.f};
      if (l < r && jj < J) {
        const float* hp = H + (int64_t)l * n + cc;
        if (cc + CPL - 1 < n) {
          if (CPL == 4) {
            const float4 h4 = *reinterpret_cast<const float4*>(hp);
            hx[0] = h4.x; hx[1] = h4.y; hx[2] = h4.z; hx[3] = h4.w;
          } else {
            const float2 h2 = *reinterpret_cast<const float2*>(hp);
            hx[0] = h2.x; hx[1] = h2.y;
          }
        } else {
#pragma unroll
          for (int t = 0; t < CPL - 1; ++t)
            if (cc + t < n) hx[t] = hp[t];
        }
      }
#pragma unroll
      for (int p2 = 0; p2 < CPL / 2; ++p2) dst[l][p2] = f2(hx[2 * p2], hx[2 * p2 + 1]);
    }
  };
  // BCD mode (PersistArgs::bcdL): row scales of H_m, 1 / L_H, output buffer
  const bool bcd = pa.bcdL != nullptr;
  float bsh[R], bq[R];
  float binvL = 0.f;
#pragma unroll
  for (int l = 0; l < R; ++l) {
    bsh[l] = (bcd && l < r) ? (float)pa.bcdS[l] : 1.f;
    bq[l] = (FOLD && l < r) ? (float)pa.bcdS[64 + l] : 0.f;
  }
  if (bcd) {
    const double L = *pa.bcdL;
    binvL = L > 0.0 ? (float)(1.0 / L) : 0.f;
  }
  float* const Ho = (bcd && pa.Hout) ? ((pa.bcdRole && *pa.bcdRole != 0.0) ? pa.Hout2 : pa.Hout) : H;
  float2 hnext[R][CPL / 2];
  if (HDIRECT) load_h(warp, hnext);

  for (int64_t j = warp; j < J; j += NWT) {
    const int64_t pos = pbase + j;
    const int64_t jt = (b + j * gridDim.x) * BNT;  // first column of the tile
    const int64_t c0 = jt + cq;
    float2 hv[R][CPL / 2];
#pragma unroll
    for (int l = 0; l < R; ++l)
#pragma unroll
      for (int p2 = 0; p2 < CPL / 2; ++p2) hv[l][p2] = HDIRECT ? hnext[l][p2] : f2(0.f, 0.f);
    if (HDIRECT) load_h(j + NWT, hnext);
    {
#ifdef NTT_WATCHDOG
      long long t0 = clock64();
#endif
      if (lane == 0) {
        while (ld_acquire_u32(issued) <= (uint32_t)pos) {
          __nanosleep(64);
#ifdef NTT_WATCHDOG
          if (clock64() - t0 > 4000000000LL) {
            printf("WATCHDOG issued block=%d warp=%d j=%lld issued=%u\n", blockIdx.x, warp, (long long)j, *issued);
            __trap();
          }
#endif
        }
      }
    }
    __syncwarp();
    const uint32_t tg = lane < ns ? *reinterpret_cast<volatile uint32_t*>(tag + lane) : 0xffffffffu;
    const unsigned hit = __ballot_sync(0xffffffffu, (tg >> 1) == (uint32_t)pos && lane < ns);
    const int s = __ffs(hit) - 1;
    const uint32_t ph = __shfl_sync(0xffffffffu, tg, s) & 1u;
    MBAR_WAIT(&full[s], ph, 2, j);
    const unsigned char* st = stages + (size_t)s * SB;
    float* Hw = HDIRECT ? HwDirect : reinterpret_cast<float*>(stages + (size_t)s * SB + XB);
    if (!HDIRECT) {
      const unsigned char* hb = st + XB + qbox * 1024;
#pragma unroll
      for (int l = 0; l < R; ++l) {
        const unsigned char* hp = hb + l * 128 + ((qch ^ l) << 4) + qsub * 4;
        if (CPL == 4) {
          const float4 h4 = lds128(hp);
          hv[l][0] = f2(h4.x, h4.y);
          hv[l][CPL / 2 - 1] = f2(h4.z, h4.w);
        } else {
          hv[l][0] = *reinterpret_cast<const float2*>(hp);
        }
      }
    }
    if (FOLD && ext) {  // H_m = a H_prev - b H_prev2 (bcd.cu k_bcd_wside, BS_FOLD)
      const unsigned char* qb = st + XB + HB + qbox * 1024;
#pragma unroll
      for (int l = 0; l < R; ++l) {
        const unsigned char* qp = qb + l * 128 + ((qch ^ l) << 4) + qsub * 4;
        float2 hq[CPL / 2];
        if (CPL == 4) {
          const float4 q4 = lds128(qp);
          hq[0] = f2(q4.x, q4.y);
          hq[CPL / 2 - 1] = f2(q4.z, q4.w);
        } else {
          hq[0] = *reinterpret_cast<const float2*>(qp);
        }
#pragma unroll
        for (int p2 = 0; p2 < CPL / 2; ++p2)
          hv[l][p2] = f2(fmaf(bsh[l], hv[l][p2].x, -bq[l] * hq[p2].x), fmaf(bsh[l], hv[l][p2].y, -bq[l] * hq[p2].y));
      }
    } else if (bcd) {  // H_m = diag(sH) H_m stored (bcd.cu's l.9 compensation)
#pragma unroll
      for (int l = 0; l < R; ++l)
#pragma unroll
        for (int p2 = 0; p2 < CPL / 2; ++p2) hv[l][p2] = f2(hv[l][p2].x * bsh[l], hv[l][p2].y * bsh[l]);
    }

    // ---------------- phase A ----------------
    {
      float2 hn[R][CPL / 2];
      if (do_update) {
        const unsigned char* xb = st + qbox * MP * 128 + qsub * 4;
        float2 s2[R][CPL / 2];
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int p2 = 0; p2 < CPL / 2; ++p2) s2[k][p2] = f2(0.f, 0.f);
#pragma unroll 4
        for (int i = 0; i < m; ++i) {
          const int offi = (qch ^ (i & 7)) << 4;
          float2 xv[CPL / 2];
          if (CPL == 4) {
            const float4 x = lds128(xb + offi + i * 128);
            xv[0] = f2(x.x, x.y);
            xv[CPL / 2 - 1] = f2(x.z, x.w);
          } else {
            xv[0] = *reinterpret_cast<const float2*>(xb + offi + i * 128);
          }
          const float4* wr = reinterpret_cast<const float4*>(Ws + i * 8);
          float w[8];
          *reinterpret_cast<float4*>(w) = wr[0];
          if (R > 4) *reinterpret_cast<float4*>(w + 4) = wr[1];
#pragma unroll
          for (int k = 0; k < R; ++k)
#pragma unroll
            for (int p2 = 0; p2 < CPL / 2; ++p2) s2[k][p2] = __ffma2_rn(bc(w[k]), xv[p2], s2[k][p2]);
        }
        // E = G H (l outer: independent accumulators) ; Hn = H S / (E + eps)
        float2 ev[R][CPL / 2];
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int p2 = 0; p2 < CPL / 2; ++p2) ev[k][p2] = f2(0.f, 0.f);
#pragma unroll
        for (int l = 0; l < R; ++l) {
          // G = W^T W is symmetric: G[k][l] = Gs[l * 8 + k], read as two 128-bit words
          float gl[8];
          *reinterpret_cast<float4*>(gl) = *reinterpret_cast<const float4*>(Gs + l * 8);
          if (R > 4) *reinterpret_cast<float4*>(gl + 4) = *reinterpret_cast<const float4*>(Gs + l * 8 + 4);
#pragma unroll
          for (int k = 0; k < R; ++k) {
            const float g = gl[k];
#pragma unroll
            for (int p2 = 0; p2 < CPL / 2; ++p2) ev[k][p2] = __ffma2_rn(bc(g), hv[l][p2], ev[k][p2]);
          }
        }
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int p2 = 0; p2 < CPL / 2; ++p2) {
            float2 v;
            if (bcd) {  // prox-linear step (Alg. 3 l.14): max(0, H_m - (G H_m - S) / L_H)
              v.x = fmaxf(0.f, fmaf(-(ev[k][p2].x - s2[k][p2].x), binvL, hv[k][p2].x));
              v.y = fmaxf(0.f, fmaf(-(ev[k][p2].y - s2[k][p2].y), binvL, hv[k][p2].y));
            } else {
              v.x = mu_q(hv[k][p2].x, s2[k][p2].x, ev[k][p2].x, eps);
              v.y = mu_q(hv[k][p2].y, s2[k][p2].y, ev[k][p2].y, eps);
            }
            if (k >= r) v = f2(0.f, 0.f);  // padded ranks (0/0 when eps = 0)
            // columns beyond n: zero (never stored, never accumulated)
            if (c0 + 2 * p2 >= n) v.x = 0.f;
            if (c0 + 2 * p2 + 1 >= n) v.y = 0.f;
            hn[k][p2] = v;
          }
        // store H (in place -- this tile's H was already read -- or to Hout for BCD)
        if (c0 + CPL - 1 < n) {
#pragma unroll
          for (int k = 0; k < R; ++k)
            if (k < r) {
              if (CPL == 4)
                *reinterpret_cast<float4*>(Ho + (int64_t)k * n + c0) =
                    make_float4(hn[k][0].x, hn[k][0].y, hn[k][CPL / 2 - 1].x, hn[k][CPL / 2 - 1].y);
              else
                *reinterpret_cast<float2*>(Ho + (int64_t)k * n + c0) = hn[k][0];
            }
        } else {
#pragma unroll
          for (int k = 0; k < R; ++k)
            if (k < r) {
#pragma unroll
              for (int t = 0; t < CPL - 1; ++t)
                if (c0 + t < n) Ho[(int64_t)k * n + c0 + t] = (t & 1) ? hn[k][t >> 1].y : hn[k][t >> 1].x;
            }
        }
      } else {
#pragma unroll
        for (int k = 0; k < R; ++k)
#pragma unroll
          for (int p2 = 0; p2 < CPL / 2; ++p2) hn[k][p2] = hv[k][p2];
      }
      if (do_acc) {
        // transposed Hn tile: Hw[hn_idx(c, k)] (HDIRECT) or over the H boxes (all lanes have read H)
        if (!HDIRECT) __syncwarp();
#pragma unroll
        for (int t = 0; t < CPL; ++t) {
          float tv[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) tv[k] = (k < R) ? ((t & 1) ? hn[k % R][t >> 1].y : hn[k % R][t >> 1].x) : 0.f;
          float* dst = Hw + (HDIRECT ? hn_idx(cq + t, 0) : hn_sw<SL>(cq + t, 0));
          *reinterpret_cast<float4*>(dst) = make_float4(tv[0], tv[1], tv[2], tv[3]);
          if (R > 4) *reinterpret_cast<float4*>(dst + 4) = make_float4(tv[4], tv[5], tv[6], tv[7]);
        }
      }
    }

    // ---------------- phase B ----------------
    if (do_acc) {
      __syncwarp();
#pragma unroll 2
      for (int s4 = 0; s4 < SL / 4; ++s4) {
        const int c = SL * cs + 4 * s4;
        const unsigned char* xb = st + (c >> 5) * MP * 128;
        const int chk = (c & 31) >> 2;
        float2 hq2[4][R / 2];
        float hq[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const float* src = Hw + (HDIRECT ? hn_idx(c + t, 0) : hn_sw<SL>(c + t, 0));
          float4 a = *reinterpret_cast<const float4*>(src);
          hq2[t][0] = f2(a.x, a.y);
          if (R > 2) hq2[t][1 % (R / 2)] = f2(a.z, a.w);
          if (R > 4) {
            float4 bq = *reinterpret_cast<const float4*>(src + 4);
            hq2[t][2 % (R / 2)] = f2(bq.x, bq.y);
            if (R > 6) hq2[t][3 % (R / 2)] = f2(bq.z, bq.w);
          }
          hq[t] = src[rb];
        }
        float xs[UX][4];
#pragma unroll
        for (int u = 0; u < UX; ++u) {
          const float4 x = lds128(xb + (rb + 8 * u) * 128 + ((chk ^ rb) << 4));
          xs[u][0] = x.x;
          xs[u][1] = x.y;
          xs[u][2] = x.z;
          xs[u][3] = x.w;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int u = 0; u < UX; ++u)
#pragma unroll
            for (int kp = 0; kp < R / 2; ++kp) acc[u * (R / 2) + kp] = __ffma2_rn(bc(xs[u][t]), hq2[t][kp], acc[u * (R / 2) + kp]);
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int kp = 0; kp < R / 2; ++kp) acc[UX * (R / 2) + kp] = __ffma2_rn(bc(hq[t]), hq2[t][kp], acc[UX * (R / 2) + kp]);
      }
      ++ntile;
    }
    if (do_acc && (ntile == RS || j + NWT >= J)) {
      ntile = 0;
      // reduce-scatter over the 4 lanes with the same rb (xor 16, then xor 8)
      float a1[V4];
#pragma unroll
      for (int v = 0; v < V4 / 2; ++v) {
        a1[2 * v] = acc[v].x;
        a1[2 * v + 1] = acc[v].y;
      }
      float a2[V4 / 2];
#pragma unroll
      for (int v = 0; v < V4 / 2; ++v) {
        const float send = h1 ? a1[v] : a1[v + V4 / 2];
        const float keep = h1 ? a1[v + V4 / 2] : a1[v];
        a2[v] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
      }
#pragma unroll
      for (int v = 0; v < V4 / 4; ++v) {
        const float send = h0 ? a2[v] : a2[v + V4 / 4];
        const float keep = h0 ? a2[v + V4 / 4] : a2[v];
        accd[v] += (double)(keep + __shfl_xor_sync(0xffffffffu, send, 8));
      }
#pragma unroll
      for (int v = 0; v < V4 / 2; ++v) acc[v] = f2(0.f, 0.f);
    }
    // Hn was written over the stage with generic stores: order them before the
    // producer's next TMA (async-proxy) write into this stage
    if (!HDIRECT && do_acc) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) asm volatile("red.release.cta.shared::cta.or.b32 [%0], %1;" ::"r"(smem_u32(free_mask)), "r"(1u << s) : "memory");
  }

  if (do_acc) {
  // ---- fixed-order CTA reduction of the per-thread fp64 partials
  asm volatile("bar.sync 1, %0;" ::"r"(NWT * 32) : "memory");
  // red[w][rb][f], f = u*R + k flat (u = UX is the Q row)
  double* red = reinterpret_cast<double*>(stages);
#pragma unroll
  for (int v = 0; v < V4 / 4; ++v) red[((size_t)warp * 8 + rb) * V4 + cs * (V4 / 4) + v] = accd[v];
  asm volatile("bar.sync 1, %0;" ::"r"(NWT * 32) : "memory");
  const int mr = m * r, rr = r * r;
  double* Pb = persist ? pa.part + b * (mr + rr) : Ppart + b * mr;
  double* Qb = persist ? pa.part + b * (mr + rr) + mr : Qpart + b * rr;
  for (int e = tid; e < 8 * V; e += NWT * 32) {
    const int rbe = e / V, f = e % V;
    const int u = f / R, k = f % R;
    if (k >= r) continue;
    const bool isQ = (u == UX);
    const int row = isQ ? rbe : rbe + 8 * u;
    if (isQ ? (row >= r) : (row >= m)) continue;
    double sum = 0.0;
    for (int w = 0; w < NWT; ++w) sum += red[((size_t)w * 8 + rbe) * V4 + f];
    if (isQ) Qb[row * r + k] = sum;
    else Pb[row * r + k] = sum;
  }
  }
  }  // consumer warps
  if (!persist || !do_acc) break;
  persist_step<8>(pa, epoch, m, r, eps, Ws, Gs, reinterpret_cast<double*>(stages), it, xs0);
  }  // passes
  if (persist) xseq_store(pa, xs0);
}



// ---------------------------------------------------------------------------
// fp16 hi/lo operand split for warp-level mma.sync (k_fused_c): v = 2^-e (hi + lo) with
// hi = fp16(v 2^e), lo = fp16(v 2^e - hi) (~22 significant bits; the lo x lo product is
// dropped), 2^e a power of two chosen per operand block so |v| 2^e < 2^14.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ void split2(float a, float b, float s, uint32_t& hi, uint32_t& lo) {
  const float2 x = __fmul2_rn(make_float2(a, b), make_float2(s, s));
  const __half2 h = __float22half2_rn(x);
  const float2 hf = __half22float2(h);
  const __half2 l = __float22half2_rn(make_float2(x.x - hf.x, x.y - hf.y));
  hi = h2_bits(h);
  lo = h2_bits(l);
}
// power-of-two scale for a block whose max |v| is mx: (2^e, 2^-e) with mx 2^e in [2^13, 2^14)
__device__ __forceinline__ float2 pow2_scale(float mx) {
  const int ex = (int)((__float_as_uint(mx) >> 23) & 255u);
  int e = ex == 0 ? 0 : 140 - ex;
  e = e < -120 ? -120 : (e > 120 ? 120 : e);
  return make_float2(__uint_as_float((uint32_t)(e + 127) << 23), __uint_as_float((uint32_t)(127 - e) << 23));
}
// max over the warp of non-negative floats: one redux.sync on the bit patterns (which order
// like the values for v >= 0)
__device__ __forceinline__ float warp_max(float v) {
  return __uint_as_float(__reduce_max_sync(0xffffffffu, __float_as_uint(v)));
}
__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
// D += A B (m16n8k16, fp16 inputs, fp32 accumulators)
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// byte offset of 16-byte chunk `ch` (0..3) of row `row` in a [rows][32] fp16 array (64-byte
// rows, chunk XOR (row / 2) mod 4: conflict-free for ldmatrix's 8-row phases)
__device__ __forceinline__ uint32_t h16_off(int row, int ch) { return (uint32_t)(row * 64 + ((ch ^ ((row >> 1) & 3)) << 4)); }

// ===========================================================================
// k_fused_c: the one-pass MU / BCD kernel for 40 < m <= 256, rank padded to RK = 8 or 16,
// on warp-level tensor cores (mma.sync m16n8k16, fp16 hi / lo splits; helpers above).
// Small CTAs (4 consumer warps + 1 TMA warp, <= 113 KB smem) so TWO CTAs share an SM and
// one CTA's serial sections (S reduction, H update, barriers) overlap the other's.  Tile =
// 32 columns x MP rows of X (one box) + the RK x 32 box of H.  Warp w owns rows
// [RW w, RW w + RW) in 32-row blocks:
//   X      -> fp16 hi / lo blocks in place (per-block scale); a persistent launch stores them
//             in the X16 cache in its prologue pass and streams them afterwards
//   phase A S^T (32 x RK) partial = X^T W over the warp's rows; fixed-order sum over the
//           warps in smem
//   H update 128 threads form E = G H and Hn (RK / 4 entries each; MU rule or BCD step)
//   phase B P (the warp's rows x RK) += X Hn^T; warp 0 adds Q += Hn Hn^T
// Rows are disjoint across warps, so per-CTA partials need no cross-warp reduction.
// ===========================================================================
constexpr int BNC = 32;
constexpr int SMEM_C = 113 * 1024;      // two CTAs per SM

// transposed Hn tile [c][k], RK floats per column + 4 floats of padding per 8 columns
template <int RK>
__device__ __forceinline__ int hnc_idx(int c, int k) { return c * RK + k + 4 * (c >> 3); }
constexpr int hnc_floats(int rk) { return 32 * rk + 16; }
// byte offset of element (k, c) of the RK x 32 H box (TMA SWIZZLE_128B: 1 KB atoms of 8 rows)
__device__ __forceinline__ int hc_off(int k, int c) { return k * 128 + ((((c >> 2) ^ k) & 7) << 4) + (c & 3) * 4; }

template <int MP, int NW, int RK>
// NW = 4: two CTAs per SM (10 warps over 4 sub-partitions: <= 3 x 32 x 170 registers in one 16 K
// bank -> 168 registers); NW = 8 (the RK = 16 class at MP = 256): one CTA per SM, <= 224 registers
__global__ void __launch_bounds__((NW + 1) * 32, NW == 4 ? 2 : 1)
k_fused_c(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmH, int m, int64_t n, int r,
          const float* __restrict__ W, const double* __restrict__ Gpart, int nG, float eps, float* __restrict__ H,
          double* __restrict__ Ppart, double* __restrict__ Qpart, int mode, int ns, int evict_first,
          PersistArgs pa) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int RW = MP / NW;           // rows per warp (32 or 64)
  constexpr int NB = RW / 32;           // 32-row blocks per warp
  constexpr int NN = RK / 8;            // n-tiles of 8 ranks
  static_assert(RW >= 32 && RW % 32 == 0, "k_fused_c: at least 32 rows per consumer warp");
  static_assert(NW == 4 || NW == 8, "k_fused_c: 4 or 8 consumer warps");
  constexpr int HH = RK / NW;           // H-update (k, c) pairs per thread
  constexpr int NTHR = (NW + 1) * 32;
  constexpr int NBAR = NW * 32;
  constexpr uint32_t XB = MP * 128u;
  constexpr uint32_t SB = XB + RK * 128u;
  unsigned char* stages = smem;
  // [NW][RK k][SRS] (32 columns + 4 floats of padding: the phase-A fragment stores (column g,
  // rank 2t) of a warp hit 32 distinct banks; a 32-float row made them 4-way conflicted)
  constexpr int SRS = 36;
  float* Sred = reinterpret_cast<float*>(smem + (size_t)ns * SB);
  float* Gs = Sred + NW * RK * SRS;                                  // RK x RK
  float* Hn = Gs + RK * RK;                                          // hnc_floats(RK)
  float* Wc = Hn + hnc_floats(RK);                                   // MP x RK (rank padded)
  uint64_t* full = reinterpret_cast<uint64_t*>(Wc + MP * RK);
  uint64_t* empty = full + ns;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool persist = pa.iters > 0;
  // BCD mode (PersistArgs::bcdL; see k_fused): row scales of H_m (smem), 1 / L_H, output buffer
  const bool bcd = pa.bcdL != nullptr;
  __shared__ float bsh[RK];
  __shared__ float hmx[NW];  // per-warp max |Hn| of the current tile (phase B scale)
  if (tid < RK) bsh[tid] = (bcd && tid < r) ? (float)pa.bcdS[tid] : 1.f;
  const float binvL = (bcd && *pa.bcdL > 0.0) ? (float)(1.0 / *pa.bcdL) : 0.f;
  float* const Ho = (bcd && pa.Hout) ? ((pa.bcdRole && *pa.bcdRole != 0.0) ? pa.Hout2 : pa.Hout) : H;
  if (!persist && (mode & kFusedUpdate)) {
    const int rr = r * r;
    for (int e = tid; e < RK * RK; e += NTHR) {
      const int k = e / RK, l = e % RK;
      double sum = 0.0;
      if (k < r && l < r)
        for (int bq = 0; bq < nG; ++bq) sum += Gpart[(int64_t)bq * rr + k * r + l];
      Gs[e] = (float)sum;
    }
  }
  for (int e = tid; e < MP * RK; e += NTHR) {
    const int i = e / RK, k = e % RK;
    Wc[e] = (i < m && k < r) ? W[(int64_t)i * r + k] : 0.0f;
  }
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t ntiles = (n + BNC - 1) / BNC;
  const int64_t b = blockIdx.x;
  const int nblk = (m + 31) / 32;                           // 32-row blocks of X present in a tile
  const int64_t x16_stride = (int64_t)nblk * 4096 + 128;   // per-tile blob: blocks + 32 scales
  const int64_t J = (ntiles > b) ? (ntiles - b + gridDim.x - 1) / gridDim.x : 0;

  unsigned epoch = 0;
  int ring_s = 0;          // ring stage / parity of the next tile (continues across passes)
  uint32_t ring_ph = 0;
  const int nit = persist ? pa.iters + 1 : 1;
  const unsigned long long xs0 = persist ? xseq_load(pa) : 0ull;
  for (int it = 0; it < nit; ++it) {
  const int md = persist ? (it == 0 ? kFusedAcc : (kFusedUpdate | (it < pa.iters ? kFusedAcc : 0))) : mode;
  const bool do_update = (md & kFusedUpdate) != 0;
  const bool do_acc = (md & kFusedAcc) != 0;
  // X16 cache: the prologue pass (it == 0) writes it, every later pass streams it
  const bool x16_write = pa.x16 != nullptr && persist && it == 0;
  const bool x16_read = pa.x16 != nullptr && persist && it > 0;
  pstamp(pa, it, 0);
  if (warp == NW) {
    if (lane == 0) {
      const uint64_t policy = evict_first ? policy_evict_first() : policy_evict_normal();
      for (int64_t j = 0; j < J; ++j) {
        const int s = ring_s;
        const uint32_t ph = ring_ph;
        if (++ring_s == ns) {
          ring_s = 0;
          ring_ph ^= 1u;
        }
        MBAR_WAIT_BACKOFF(&empty[s], ph ^ 1u, 3, j);
        const int64_t tile = b + j * gridDim.x;
        const int col0 = (int)(tile * BNC);
        unsigned char* st = stages + (size_t)s * SB;
        if (x16_read) {  // the tile's fp16 hi / lo blocks, one contiguous bulk copy
          NTT_DCHECK(tile < ntiles);
          mbar_expect_tx(&full[s], (uint32_t)(nblk * 4096) + RK * 128u);
          bulk_load_1d(st, pa.x16 + tile * x16_stride, (uint32_t)(nblk * 4096), &full[s], policy);
        } else {
          mbar_expect_tx(&full[s], SB);
          tma_load_2d(st, &tmX, col0, 0, &full[s], policy);
        }
        tma_load_2d(st + XB, &tmH, col0, 0, &full[s], policy);
      }
    }
  } else {

  // One pass's tile loop, instantiated per pass mode (UPD: phase A + H update, ACC: phase B,
  // BCD: Alg. 3's prox-linear H step instead of the MU rule), so no per-tile branch on the mode.
  auto pass_tiles = [&](auto upd_t, auto acc_t, auto bcd_t) {
  constexpr bool UPD = decltype(upd_t)::value, ACC = decltype(acc_t)::value, BCD = decltype(bcd_t)::value;
  const int fg = lane >> 2, ft = lane & 3;  // mma fragment coordinates (group, thread in group)
  float xsi[NB];               // 2^-e of each block's X split (this tile)
#pragma unroll
  for (int bb = 0; bb < NB; ++bb) xsi[bb] = 1.f;
  // phase A's B operand: W rows of this warp as fp16 hi / lo fragments, one scale per warp and pass:
  // b0 = {W[r0 + 2ft][8nn + fg], W[r0 + 2ft + 1][..]}, b1 = rows + 8, + 9; r0 = warp RW + 32 bb + 16 ks
  uint32_t wfh[NB][2][NN][2], wfl[NB][2][NN][2];
  float wsi = 1.f;
  if constexpr (UPD) {
    float wm = 0.f;
#pragma unroll
    for (int bb = 0; bb < NB; ++bb)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int nn = 0; nn < NN; ++nn)
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int r0 = warp * RW + 32 * bb + 16 * ks + 8 * h2 + 2 * ft, k = 8 * nn + fg;
            wm = fmaxf(wm, fmaxf(fabsf(Wc[r0 * RK + k]), fabsf(Wc[(r0 + 1) * RK + k])));
          }
    const float2 wsc = pow2_scale(warp_max(wm));
    wsi = wsc.y;
#pragma unroll
    for (int bb = 0; bb < NB; ++bb)
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int nn = 0; nn < NN; ++nn)
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            const int r0 = warp * RW + 32 * bb + 16 * ks + 8 * h2 + 2 * ft, k = 8 * nn + fg;
            split2(Wc[r0 * RK + k], Wc[(r0 + 1) * RK + k], wsc.x, wfh[bb][ks][nn][h2], wfl[bb][ks][nn][h2]);
          }
  }
  // two-level P accumulation (fp32 over <= 8 tiles, then fp64); RK = 16 adds each tile's fp32 sum to
  // fp64 directly (the fp32 set would not fit in 200 registers next to the fp64 one)
  constexpr bool P32 = false;  // RK = 8 too: the fp32 level cost 16 registers and 72 B of spills in the tile loop
  float pacc[P32 ? NB : 1][2][NN][4];
  double paccd[NB][2][NN][4];
  // Q = Hn Hn^T.  RK = 16: on mma.sync by warp 0 (the A fragments of Hn are phase B's B
  // fragments; 7 % faster at 256 x 2^24, r 10, than 48 shared loads per thread and tile), fp64
  // accumulation per tile, rows fg (+ 8), ranks 8 nn + 2 ft (+ 1).  RK = 8: FFMA over column
  // slices (the mma form's registers cost 76 B of spills and 4 % in <256,4,8>)
  constexpr bool QMMA = RK == 16;
  constexpr int QR = RK / NW;  // Q rows per warp (FFMA form)
  double qdd[QMMA ? NN : 1][4];
  double qd[QMMA ? 1 : QR];
#pragma unroll
  for (int qq = 0; qq < (QMMA ? 1 : QR); ++qq) qd[qq] = 0.0;
#pragma unroll
  for (int bb = 0; bb < NB; ++bb)
#pragma unroll
    for (int mh = 0; mh < 2; ++mh)
#pragma unroll
      for (int nn = 0; nn < NN; ++nn)
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          if constexpr (P32) pacc[bb][mh][nn][e4] = 0.f;
          paccd[bb][mh][nn][e4] = 0.0;
        }
#pragma unroll
  for (int nn = 0; nn < (QMMA ? NN : 1); ++nn)
#pragma unroll
    for (int e4 = 0; e4 < 4; ++e4) qdd[nn][e4] = 0.0;
  int since_flush = 0;
  // X16 passes: the block scales of a tile (written by the prologue pass next to its blocks, read
  // from L2) are loaded one tile ahead -- on the critical path they cost an L2 round trip per tile
  float xsn[NB];
  auto load_scales = [&](int64_t jj) {
    const float* sc = reinterpret_cast<const float*>(pa.x16 + (b + jj * gridDim.x) * x16_stride + nblk * 4096);
#pragma unroll
    for (int bb = 0; bb < NB; ++bb) {
      const int gb = warp * NB + bb;
      xsn[bb] = gb < nblk ? __ldcg(sc + gb) : 0.f;
    }
  };
  if (x16_read && J > 0) load_scales(0);

  for (int64_t j = 0; j < J; ++j) {
    const int s = ring_s;
    const uint32_t ph = ring_ph;
    if (++ring_s == ns) {
      ring_s = 0;
      ring_ph ^= 1u;
    }
    NTT_DCHECK(s >= 0 && s < ns);
    MBAR_WAIT(&full[s], ph, 4, j);
    unsigned char* st = stages + (size_t)s * SB;
    const unsigned char* hbox = st + XB;
    const int64_t jt = (b + j * gridDim.x) * BNC;

    if constexpr (!UPD) {
      // prologue: Hn of the previous tile may still be read by phase B of other warps
      asm volatile("bar.sync 1, %0;" ::"r"(NBAR) : "memory");
    }
    if (x16_read) {
#pragma unroll
      for (int bb = 0; bb < NB; ++bb) xsi[bb] = xsn[bb];
      if (j + 1 < J) load_scales(j + 1);
    } else {
      // ---- this warp's rows of the tile -> fp16 hi / lo parts, in place (each 32-row block of
      // 4 KB fp32 becomes [hi: 32 x 32 fp16 | lo: 32 x 32 fp16]); per-block power-of-two scale;
      // the prologue pass of a persistent launch also stores them to the X16 cache
      unsigned char* gtile = x16_write ? pa.x16 + (b + j * gridDim.x) * x16_stride : nullptr;
#pragma unroll
      for (int bb = 0; bb < NB; ++bb) {
        const int gb = warp * NB + bb;
        unsigned char* blk = st + (size_t)(warp * RW + 32 * bb) * 128;
        float v[32];
#pragma unroll
        for (int c16 = 0; c16 < 8; ++c16) {
          const float4 f = lds128(blk + lane * 128 + ((c16 ^ (lane & 7)) << 4));
          v[4 * c16] = f.x;
          v[4 * c16 + 1] = f.y;
          v[4 * c16 + 2] = f.z;
          v[4 * c16 + 3] = f.w;
        }
        float m8[8];  // max |v| as a tree (depth 4) rather than a 31-long chain
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2)
          m8[q2] = fmaxf(fmaxf(fabsf(v[4 * q2]), fabsf(v[4 * q2 + 1])), fmaxf(fabsf(v[4 * q2 + 2]), fabsf(v[4 * q2 + 3])));
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        const float2 sc = pow2_scale(warp_max(mx));
        xsi[bb] = sc.y;
        __syncwarp();
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          uint32_t hh[4], ll[4];
#pragma unroll
          for (int p2 = 0; p2 < 4; ++p2) split2(v[8 * k4 + 2 * p2], v[8 * k4 + 2 * p2 + 1], sc.x, hh[p2], ll[p2]);
          *reinterpret_cast<uint4*>(blk + h16_off(lane, k4)) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
          *reinterpret_cast<uint4*>(blk + 2048 + h16_off(lane, k4)) = make_uint4(ll[0], ll[1], ll[2], ll[3]);
          if (gtile && gb < nblk) {
            __stcg(reinterpret_cast<uint4*>(gtile + gb * 4096 + h16_off(lane, k4)), make_uint4(hh[0], hh[1], hh[2], hh[3]));
            __stcg(reinterpret_cast<uint4*>(gtile + gb * 4096 + 2048 + h16_off(lane, k4)),
                   make_uint4(ll[0], ll[1], ll[2], ll[3]));
          }
        }
        if (gtile && gb < nblk && lane == 0) __stcg(reinterpret_cast<float*>(gtile + nblk * 4096) + gb, sc.y);
      }
      __syncwarp();
    }
    if constexpr (UPD) {
      // ---- phase A: S^T (32 cols x RK) = X^T W over this warp's rows: A = X^T (ldmatrix.trans
      // of the fp16 parts), B = W fragments, hi.hi + hi.lo + lo.hi
      float sacc[2][NN][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nn = 0; nn < NN; ++nn)
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) sacc[mt][nn][e4] = 0.f;
#pragma unroll
      for (int bb = 0; bb < NB; ++bb) {
        // blocks of rows >= m are not loaded by the X16 passes (stale shared memory): skip them
        if (warp * NB + bb >= nblk) continue;
        const uint32_t blk = smem_u32(st) + (uint32_t)(warp * RW + 32 * bb) * 128u;
        float dacc[2][NN][4];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nn = 0; nn < NN; ++nn)
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) dacc[mt][nn][e4] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
          for (int mt = 0; mt < 2; ++mt) {
            const int mj = lane >> 3;
            const uint32_t off = h16_off(16 * ks + (lane & 7) + 8 * (mj >> 1), 2 * mt + (mj & 1));
            uint32_t ah[4], al[4];
            ldsm_x4_t(blk + off, ah);
            ldsm_x4_t(blk + 2048u + off, al);
#pragma unroll
            for (int nn = 0; nn < NN; ++nn) {
              mma16816(dacc[mt][nn], ah, wfh[bb][ks][nn][0], wfh[bb][ks][nn][1]);
              mma16816(dacc[mt][nn], ah, wfl[bb][ks][nn][0], wfl[bb][ks][nn][1]);
              mma16816(dacc[mt][nn], al, wfh[bb][ks][nn][0], wfh[bb][ks][nn][1]);
            }
          }
        const float f = xsi[bb] * wsi;
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
          for (int nn = 0; nn < NN; ++nn)
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) sacc[mt][nn][e4] = fmaf(dacc[mt][nn][e4], f, sacc[mt][nn][e4]);
      }
      // fragment (col 16 mt + fg (+8 for e4 >= 2), rank 8 nn + 2 ft + (e4 & 1)) -> Sred[w][rank][col]
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int nn = 0; nn < NN; ++nn)
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4)
            Sred[(warp * RK + 8 * nn + 2 * ft + (e4 & 1)) * SRS + 16 * mt + fg + 8 * (e4 >> 1)] = sacc[mt][nn][e4];
      asm volatile("bar.sync 1, %0;" ::"r"(NBAR) : "memory");
    }
    // ---- H update: thread handles (k, c) for k = kt + NW hh, c = ct
    float hmax = 0.f;
    {
      const int ct = tid & 31;
      const int64_t col = jt + ct;
      float hl[RK];
#pragma unroll
      for (int l = 0; l < RK; ++l) hl[l] = *reinterpret_cast<const float*>(hbox + hc_off(l, ct));
#pragma unroll
      for (int hh = 0; hh < HH; ++hh) {
        const int kt = (tid >> 5) + NW * hh;
        const float hkc = *reinterpret_cast<const float*>(hbox + hc_off(kt, ct));  // not hl[kt]: a run-time index would put hl in local memory
        float hn;
        if constexpr (UPD) {
          float S = 0.0f;
#pragma unroll
          for (int w = 0; w < NW; ++w) S += Sred[(w * RK + kt) * SRS + ct];
          float e0 = 0.0f, e1 = 0.0f;
          const float4* g4 = reinterpret_cast<const float4*>(Gs + kt * RK);  // row kt, 128-bit loads
#pragma unroll
          for (int l4 = 0; l4 < RK / 4; ++l4) {
            const float4 g = g4[l4];
            const int l = 4 * l4;
            e0 = fmaf(g.x, BCD ? hl[l] * bsh[l] : hl[l], e0);
            e1 = fmaf(g.y, BCD ? hl[l + 1] * bsh[l + 1] : hl[l + 1], e1);
            e0 = fmaf(g.z, BCD ? hl[l + 2] * bsh[l + 2] : hl[l + 2], e0);
            e1 = fmaf(g.w, BCD ? hl[l + 3] * bsh[l + 3] : hl[l + 3], e1);
          }
          if constexpr (BCD)  // prox-linear step (Alg. 3 l.14) on H_m = diag(sH) H_m stored
            hn = fmaxf(0.f, fmaf(-((e0 + e1) - S), binvL, hkc * bsh[kt]));
          else
            hn = mu_q(hkc, S, e0 + e1, eps);
          if (kt >= r || col >= n) hn = 0.0f;
          if (kt < r && col < n) {
            NTT_DCHECK((int64_t)kt * n + col < (int64_t)r * n);
            Ho[(int64_t)kt * n + col] = hn;
          }
        } else {
          hn = (kt < r && col < n) ? hkc : 0.0f;
        }
        if constexpr (ACC) Hn[hnc_idx<RK>(ct, kt)] = hn;
        hmax = fmaxf(hmax, fabsf(hn));
      }
    }
    if constexpr (ACC) {
      const float wm = warp_max(hmax);
      if (lane == 0) hmx[warp] = wm;
      asm volatile("bar.sync 1, %0;" ::"r"(NBAR) : "memory");
      // B = Hn^T fragments, split with the tile's power-of-two scale: b0 = Hn[8 nn + g][16 kk + 2t, + 1],
      // b1 = columns + 8, + 9
      float hm = hmx[0];
#pragma unroll
      for (int w = 1; w < NW; ++w) hm = fmaxf(hm, hmx[w]);
      const float2 hsc = pow2_scale(hm);
      uint32_t bh[2][NN][2], bl[2][NN][2];
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
#pragma unroll
        for (int nn = 0; nn < NN; ++nn) {
          const int c0 = 16 * kk + 2 * ft, kr = 8 * nn + fg;
          split2(Hn[hnc_idx<RK>(c0, kr)], Hn[hnc_idx<RK>(c0 + 1, kr)], hsc.x, bh[kk][nn][0], bl[kk][nn][0]);
          split2(Hn[hnc_idx<RK>(c0 + 8, kr)], Hn[hnc_idx<RK>(c0 + 9, kr)], hsc.x, bh[kk][nn][1], bl[kk][nn][1]);
        }
      // P (this warp's rows x RK) += X Hn^T: A = X (ldmatrix of the fp16 parts)
#pragma unroll
      for (int bb = 0; bb < NB; ++bb) {
        if (warp * NB + bb >= nblk) continue;  // rows >= m (see phase A)
        const uint32_t blk = smem_u32(st) + (uint32_t)(warp * RW + 32 * bb) * 128u;
        const float f = xsi[bb] * hsc.y;
#pragma unroll
        for (int mh = 0; mh < 2; ++mh) {
          float d[NN][4];
#pragma unroll
          for (int nn = 0; nn < NN; ++nn)
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) d[nn][e4] = 0.f;
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int mj = lane >> 3;
            const uint32_t off = h16_off(16 * mh + (lane & 7) + 8 * (mj & 1), 2 * kk + (mj >> 1));
            uint32_t ah[4], al[4];
            ldsm_x4(blk + off, ah);
            ldsm_x4(blk + 2048u + off, al);
#pragma unroll
            for (int nn = 0; nn < NN; ++nn) {
              mma16816(d[nn], ah, bh[kk][nn][0], bh[kk][nn][1]);
              mma16816(d[nn], ah, bl[kk][nn][0], bl[kk][nn][1]);
              mma16816(d[nn], al, bh[kk][nn][0], bh[kk][nn][1]);
            }
          }
#pragma unroll
          for (int nn = 0; nn < NN; ++nn)
#pragma unroll
            for (int e4 = 0; e4 < 4; ++e4) {
              if constexpr (P32) pacc[bb][mh][nn][e4] = fmaf(d[nn][e4], f, pacc[bb][mh][nn][e4]);
              else paccd[bb][mh][nn][e4] += (double)(d[nn][e4] * f);
            }
        }
      }
      if constexpr (!QMMA) {  // Q rows QR w + qq, column qc = lane % RK, over this lane's slice of
                              // the tile's columns (32 / RK slices); slices summed at the end of the pass
        float qa[QR];
#pragma unroll
        for (int qq = 0; qq < QR; ++qq) qa[qq] = 0.f;
        const int qc = lane % RK, qs = lane / RK;
#pragma unroll
        for (int t = 0; t < RK; ++t) {
          const int c = qs * RK + t;
          const float hr = Hn[hnc_idx<RK>(c, qc)];
#pragma unroll
          for (int qq = 0; qq < QR; ++qq) qa[qq] = fmaf(Hn[hnc_idx<RK>(c, QR * warp + qq)], hr, qa[qq]);
        }
#pragma unroll
        for (int qq = 0; qq < QR; ++qq) qd[qq] += (double)qa[qq];
      } else if (warp == 0) {  // Q += Hn Hn^T: A = Hn (ranks x columns) = the B fragments read as A
        const float q2 = hsc.y * hsc.y;
#pragma unroll
        for (int nq = 0; nq < NN; ++nq) {
          float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const uint32_t ah[4] = {bh[kk][0][0], NN > 1 ? bh[kk][NN - 1][0] : 0u, bh[kk][0][1],
                                    NN > 1 ? bh[kk][NN - 1][1] : 0u};
            const uint32_t al[4] = {bl[kk][0][0], NN > 1 ? bl[kk][NN - 1][0] : 0u, bl[kk][0][1],
                                    NN > 1 ? bl[kk][NN - 1][1] : 0u};
            mma16816(d, ah, bh[kk][nq][0], bh[kk][nq][1]);
            mma16816(d, ah, bl[kk][nq][0], bl[kk][nq][1]);
            mma16816(d, al, bh[kk][nq][0], bh[kk][nq][1]);
          }
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) qdd[QMMA ? nq : 0][e4] += (double)(d[e4] * q2);
        }
      }
      if (P32 && ++since_flush == 8) {  // two-level accumulation: fp32 over <= 8 tiles, then fp64
        since_flush = 0;
#pragma unroll
        for (int bb = 0; bb < NB; ++bb)
#pragma unroll
          for (int mh = 0; mh < 2; ++mh)
#pragma unroll
            for (int nn = 0; nn < NN; ++nn)
#pragma unroll
              for (int e4 = 0; e4 < 4; ++e4) {
                if constexpr (P32) {
                  paccd[bb][mh][nn][e4] += (double)pacc[bb][mh][nn][e4];
                  pacc[bb][mh][nn][e4] = 0.f;
                }
              }
      }
    } else if constexpr (UPD) {
      // no phase B: the next tile's phase A must not overwrite Sred while it is still read
      asm volatile("bar.sync 1, %0;" ::"r"(NBAR) : "memory");
    }
    // the in-place X conversion wrote the stage with generic stores: order them before the
    // producer's next TMA (async-proxy) write into it
    if (!x16_read) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  if constexpr (ACC) {
    const int mr = m * r, rr = r * r;
    double* Pb = persist ? pa.part + b * (mr + rr) : Ppart + b * mr;
    double* Qb = persist ? pa.part + b * (mr + rr) + mr : Qpart + b * rr;
    // P fragment: rows warp RW + 32 bb + 16 mh + fg (+ 8), ranks 8 nn + 2 ft (+ 1)
#pragma unroll
    for (int bb = 0; bb < NB; ++bb)
#pragma unroll
      for (int mh = 0; mh < 2; ++mh)
#pragma unroll
        for (int nn = 0; nn < NN; ++nn)
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const int row = warp * RW + 32 * bb + 16 * mh + fg + 8 * (e4 >> 1), k = 8 * nn + 2 * ft + (e4 & 1);
            if (row < m && k < r) Pb[row * r + k] = paccd[bb][mh][nn][e4] + (P32 ? (double)pacc[P32 ? bb : 0][mh][nn][e4] : 0.0);
          }
    if constexpr (QMMA) {  // Q fragment (warp 0): rank rows fg (+ 8), rank columns 8 nn + 2 ft (+ 1)
      if (warp == 0)
#pragma unroll
        for (int nn = 0; nn < NN; ++nn)
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const int row = fg + 8 * (e4 >> 1), k = 8 * nn + 2 * ft + (e4 & 1);
            if (row < r && k < r) Qb[row * r + k] = qdd[QMMA ? nn : 0][e4];
          }
    } else {  // Q rows QR w + qq, column lane % RK: sum the 32 / RK column slices
#pragma unroll
      for (int qq = 0; qq < QR; ++qq) {
        qd[qq] += __shfl_xor_sync(0xffffffffu, qd[qq], 16);
        if (RK == 8) qd[qq] += __shfl_xor_sync(0xffffffffu, qd[qq], 8);
        const int row = QR * warp + qq, k = lane % RK;
        if (lane < RK && row < r && k < r) Qb[row * r + k] = qd[qq];
      }
    }
  }
  };  // pass_tiles
  using T_ = std::true_type;
  using F_ = std::false_type;
  if (!do_update) pass_tiles(F_{}, T_{}, F_{});
  else if (do_acc) bcd ? pass_tiles(T_{}, T_{}, T_{}) : pass_tiles(T_{}, T_{}, F_{});
  else bcd ? pass_tiles(T_{}, F_{}, T_{}) : pass_tiles(T_{}, F_{}, F_{});
  }  // consumer warps
  if (!persist || !do_acc) break;
  persist_step<RK>(pa, epoch, m, r, eps, Wc, Gs, reinterpret_cast<double*>(stages), it, xs0);
  }  // passes
  if (persist) xseq_store(pa, xs0);
}

// shared-memory scratch persist_step takes from the stage area between passes
size_t persist_scratch_bytes(int64_t m, int r, int rk, int threads) {
  // the slice reduction's [C][ne] partials (<= threads doubles) also live in the scratch
  int64_t d = persist_scratch_doubles(m, r, rk, threads);
  if (d < threads) d = threads;
  return sizeof(double) * (size_t)d;
}

size_t fixed_bytes_c(int MP, int NW, int RK) {
  return (size_t)NW * RK * 36 * 4 + RK * RK * 4 + hnc_floats(RK) * 4 + (size_t)MP * RK * 4 + 2 * 16 * 8 + 1024;
}

int stages_c(int MP, int NW, int RK) {
  const size_t SB = (size_t)MP * 128 + RK * 128;
  int ns = (int)(((NW == 4 ? SMEM_C : SMEM_BUDGET) - fixed_bytes_c(MP, NW, RK)) / SB);
  return ns > 12 ? 12 : ns;
}

// cooperative launch (all CTAs co-resident) for the persistent mode, plain otherwise
template <typename... KArgs, typename... Args>
cudaError_t launch_maybe_coop(void (*kern)(KArgs...), int grid, int threads, size_t smem, cudaStream_t st,
                              bool coop, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3((unsigned)threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = coop ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <int MP, int NW, int RK>
cudaError_t launch_c(const CUtensorMap& mx, const CUtensorMap& mh, int m, int64_t n, int r, const float* W,
                     const double* Gpart, int nG, float eps, float* H, double* Ppart, double* Qpart, int mode, int grid,
                     int evict_first, const PersistArgs& pa, cudaStream_t st) {
  const int ns = stages_c(MP, NW, RK);
  const size_t SB = (size_t)MP * 128 + RK * 128;
  const size_t smem = (size_t)ns * SB + fixed_bytes_c(MP, NW, RK);
  if (ns < 2) return cudaErrorInvalidConfiguration;
  if (pa.iters > 0 && persist_scratch_bytes(m, r, RK, (NW + 1) * 32) > (size_t)ns * SB) return cudaErrorInvalidConfiguration;
  cudaError_t e = smem_optin((const void*)(k_fused_c<MP, NW, RK>), smem);
  if (e != cudaSuccess) return e;
  return launch_maybe_coop(k_fused_c<MP, NW, RK>, grid, (NW + 1) * 32, smem, st, pa.iters > 0, mx, mh, m, n, r, W,
                           Gpart, nG, eps, H, Ppart, Qpart, mode, ns, evict_first, pa);
}

// ---------------------------------------------------------------- host side
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

cudaError_t get_encode() {
  if (g_encode) return cudaSuccess;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess) return e;
  if (q != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return cudaSuccess;
}

cudaError_t make_map(CUtensorMap* map, const float* base, uint64_t cols, uint64_t rows, uint64_t ld_elems,
                     uint32_t box_rows) {
  cudaError_t e = get_encode();
  if (e != cudaSuccess) return e;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * sizeof(float)};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

// X as {32 cols, rows, n / 32 column blocks} (block stride 128 B): a box {32, rows, blocks}
// lands in shared memory exactly as `blocks` 2-D boxes of 32 columns (same 128B swizzle,
// rows = 8), but as ONE transaction -- config 4's 8-row boxes are 1 KB each, in the
// small-transaction regime of the TMA engine (tools/tmabench.cu: 1 KB segments stream at
// well under half the rate of 4 KB ones).  Requires n % 32 == 0.
cudaError_t make_map3(CUtensorMap* map, const float* base, uint64_t cols, uint64_t rows, uint64_t ld_elems,
                      uint32_t box_rows, uint32_t blocks) {
  cudaError_t e = get_encode();
  if (e != cudaSuccess) return e;
  cuuint64_t dims[3] = {32, rows, cols / 32};
  cuuint64_t strides[2] = {ld_elems * sizeof(float), 32 * sizeof(float)};
  cuuint32_t box[3] = {32, box_rows, blocks};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

int ux_for(int64_t m) { return m <= 8 ? 1 : m <= 16 ? 2 : m <= 32 ? 4 : 5; }
int rcls_for(int r) { return r <= 2 ? 2 : r <= 4 ? 4 : r <= 6 ? 6 : 8; }

size_t fixed_bytes(int ux, int nwt, bool hd) {
  return (size_t)ux * 8 * 8 * 4 + 256 + (hd ? (size_t)nwt * HN_FLOATS * 4 : 0) + 2 * 24 * 8 + 160 + 1024;
}

int stages_for(int ux, int nwt, bool hd, int bnt) {
  const size_t SB = (size_t)(bnt / 32) * ux * 8 * 128 + (hd ? 0 : (size_t)(bnt / 32) * 1024);
  int ns = (int)((SMEM_BUDGET - fixed_bytes(ux, nwt, hd)) / SB);
  if (ns > 24) ns = 24;
  return ns;
}

template <int R, int UX, int NWT, bool HD, int BNT, bool FOLD = false>
cudaError_t launch_t(const CUtensorMap& mx, const CUtensorMap& mh, int m, int64_t n, int r, const float* W,
                     const double* Gpart, int nG, float eps, float* H, double* Ppart, double* Qpart, int mode, int grid,
                     int evict_first, const PersistArgs& pa, cudaStream_t st, const CUtensorMap* mh2 = nullptr) {
  const size_t HBs = HD ? 0 : (size_t)(BNT / 32) * 1024;
  const size_t SB = (size_t)(BNT / 32) * UX * 8 * 128 + HBs * (FOLD ? 2 : 1);
  int ns = FOLD ? (int)((SMEM_BUDGET - fixed_bytes(UX, NWT, HD)) / SB) : stages_for(UX, NWT, HD, BNT);
  if (ns > 24) ns = 24;
  const size_t smem = (size_t)ns * SB + fixed_bytes(UX, NWT, HD);
  if (pa.iters > 0 && persist_scratch_bytes(m, r, 8, (NWT + 1) * 32) > (size_t)ns * SB) return cudaErrorInvalidConfiguration;
  cudaError_t e = smem_optin((const void*)(k_fused<R, UX, NWT, HD, BNT, FOLD>), smem);
  if (e != cudaSuccess) return e;
  return launch_maybe_coop(k_fused<R, UX, NWT, HD, BNT, FOLD>, grid, (NWT + 1) * 32, smem, st, pa.iters > 0, mx, mh,
                           mh2 ? *mh2 : mh, m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, ns, evict_first, pa);
}

// ===========================================================================
// k_fused_m: the one-pass MU kernel for 16 < m <= 32 (rank <= 8; config 3 step 1, config 4
// steps 2-9) with all three contractions on warp-level tensor cores (mma.sync m16n8k16,
// fp16 hi / lo operand splits as in k_fused_c).  Structure as k_fused: one CTA per SM, a
// TMA producer warp with dynamic stage assignment, 8 consumer warps that each own whole
// 128-column tiles (no CTA barriers in the loop).  Per tile (lane fragment coordinates
// g = lane / 4, t = lane % 4; "mt" = 16-column m-tile):
//   E^T = H^T G      8 m-tiles x (A = H^T split in registers, B = G)      (MU denominator)
//   S^T = X^T W      8 m-tiles x 2 k-steps (A = X^T by ldmatrix.trans)     (phase A)
//   Hn  = H S / (E + eps) elementwise in the fragment layout, stored to H and over the
//         stage's H boxes
//   P  += X Hn^T     2 m-tiles x 8 k-steps (A = X by ldmatrix, B = Hn^T)    (phase B)
//   Q  += Hn Hn^T    8 k-steps (A = B = the Hn fragments)
// X is converted to fp16 hi / lo blocks in place (per 32 x 32 block scale); a persistent
// launch stores them in the X16 cache in its prologue pass and streams them afterwards.
// ===========================================================================
constexpr int NWM = 8;                     // consumer warps
constexpr int kTailGroup = 16;             // dynamic-tail claim unit (tiles; a multiple of NWM)
constexpr int XBM = 4 * 32 * 128;          // X region: 4 boxes of 32 rows x 32 columns (fp32 / fp16 hi+lo)
constexpr int HBM = 4 * 8 * 128;           // H region: 4 boxes of 8 ranks x 32 columns
constexpr int SBM = XBM + HBM + 1024;      // + 16 B of block scales (1024-aligned stages)
constexpr int X16M_STRIDE = XBM + 128;     // X16 blob per tile: 4 blocks + 4 scales

// byte offset of element (k, c) (rank k < 8, column c < 128) of the H region (TMA SWIZZLE_128B)
__device__ __forceinline__ int hbox_off(int k, int c) { return (c >> 5) * 1024 + k * 128 + ((((c & 31) >> 2) ^ k) << 4) + (c & 3) * 4; }

__global__ void __launch_bounds__((NWM + 1) * 32, 1)
k_fused_m(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmH, int m, int64_t n, int r,
          const float* __restrict__ W, const double* __restrict__ Gpart, int nG, float eps, float* __restrict__ H,
          double* __restrict__ Ppart, double* __restrict__ Qpart, int mode, int ns, int evict_first, PersistArgs pa) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int NTHR = (NWM + 1) * 32;
  unsigned char* stages = smem;
  float* Ws = reinterpret_cast<float*>(smem + (size_t)ns * SBM);  // 32 x 8
  float* Gs = Ws + 32 * 8;                                          // 8 x 8
  uint64_t* full = reinterpret_cast<uint64_t*>(Gs + 64);
  uint64_t* empty = full + ns;
  uint32_t* issued = reinterpret_cast<uint32_t*>(empty + ns);
  uint32_t* free_mask = issued + 1;
  uint32_t* tag = issued + 2;  // [ns <= 24]
  uint32_t* ptot = tag + 24;   // [2] dynamic tail: absolute end position of the pass, by parity
  int32_t* tileid = reinterpret_cast<int32_t*>(tag + 26);  // [ns <= 24] tile held by the stage
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool persist = pa.iters > 0;

  for (int e = tid; e < 32 * 8; e += NTHR) {
    const int i = e >> 3, k = e & 7;
    Ws[e] = (i < m && k < r) ? W[(int64_t)i * r + k] : 0.0f;
  }
  if (!persist && (mode & kFusedUpdate)) {
    const int rr = r * r;
    for (int e = tid; e < 64; e += NTHR) {
      const int k = e >> 3, l = e & 7;
      double s = 0.0;
      if (k < r && l < r)
        for (int q = 0; q < nG; ++q) s += Gpart[(int64_t)q * rr + k * r + l];
      Gs[e] = (float)s;
    }
  }
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    *issued = 0u;
    *free_mask = (ns >= 32) ? 0xffffffffu : ((1u << ns) - 1u);
    for (int q = 0; q < ns; ++q) tag[q] = 0xffffffffu;
    ptot[0] = ptot[1] = 0xffffffffu;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t par_mask = 0u;

  const int64_t ntiles = (n + 127) / 128;
  const int64_t b = blockIdx.x;
  const int G = gridDim.x;
  // static tiles [0, S) round robin; the dynamic tail [S, ntiles) = TG groups of kTailGroup (persistent)
  const int TG = persist ? pa.tail_groups : 0;
  const int64_t S = ntiles - kTailGroup * (int64_t)TG;
  const int64_t J = (S > b) ? (S - b + G - 1) / G : 0;  // static tiles of this CTA
  const int64_t Jmax = J + kTailGroup * (int64_t)TG;      // positions per pass (unique across passes)
  unsigned long long* pool = reinterpret_cast<unsigned long long*>(pa.ctr + 8);
  unsigned epoch = 0;
  const int nit = persist ? pa.iters + 1 : 1;
  const unsigned long long xs0 = persist ? xseq_load(pa) : 0ull;
  for (int it = 0; it < nit; ++it) {
  const int md = persist ? (it == 0 ? kFusedAcc : (kFusedUpdate | (it < pa.iters ? kFusedAcc : 0))) : mode;
  const bool do_update = (md & kFusedUpdate) != 0;
  const bool do_acc = (md & kFusedAcc) != 0;
  const bool x16_write = pa.x16 != nullptr && persist && it == 0;
  const bool x16_read = pa.x16 != nullptr && persist && it > 0;
  const int64_t pbase = (int64_t)it * Jmax;
  pstamp(pa, it, 0);
  if (warp == NWM) {
    // ================= producer =================
    if (lane == 0) {
      const uint64_t policy = evict_first ? policy_evict_first() : policy_evict_normal();
      if (TG > 0) ptot[(it + 1) & 1] = 0xffffffffu;  // the next pass's total; nobody reads it now
      auto issue = [&](const int64_t tile, const int64_t pos) {
        uint32_t fm;
        while ((fm = ld_acquire_u32(free_mask)) == 0u) __nanosleep(32);
        const int s = __ffs(fm) - 1;
        atomicAnd(free_mask, ~(1u << s));
        const uint32_t ph = (par_mask >> s) & 1u;
        par_mask ^= 1u << s;
        tag[s] = ((uint32_t)pos << 1) | ph;
        tileid[s] = (int32_t)tile;
        unsigned char* st = stages + (size_t)s * SBM;
        if (x16_read) {
          NTT_DCHECK(tile < ntiles);
          mbar_expect_tx(&full[s], XBM + HBM + 16);
          const unsigned char* src = pa.x16 + tile * X16M_STRIDE;
          bulk_load_1d(st, src, XBM, &full[s], policy);
          bulk_load_1d(st + XBM + HBM, src + XBM, 16, &full[s], policy);
        } else {
          mbar_expect_tx(&full[s], XBM + HBM);
          tma_load_3d(st, &tmX, 0, 0, (int)(tile * 4), &full[s], policy);
        }
        tma_load_3d(st + XBM, &tmH, 0, 0, (int)(tile * 4), &full[s], policy);
        st_release_u32(issued, (uint32_t)(pos + 1));
      };
      for (int64_t j = 0; j < J; ++j) issue(b + j * G, pbase + j);
      if (TG > 0) {
        // claims of this pass are [it (TG + G), (it + 1) (TG + G)): TG succeed, each CTA fails once
        const unsigned long long base = (unsigned long long)it * (unsigned long long)(TG + G);
        int64_t k = 0;
        for (;;) {
          const long long g = (long long)(atomicAdd(pool, 1ull) - base);
          if (g >= TG) break;
          for (int u = 0; u < kTailGroup; ++u) issue(S + kTailGroup * g + u, pbase + J + kTailGroup * k + u);
          ++k;
        }
        st_release_u32(&ptot[it & 1], (uint32_t)(pbase + J + kTailGroup * k));
      }
    }
  } else {
  // ================= consumer warps =================
  auto pass_tiles = [&](auto upd_t, auto acc_t) {
  constexpr bool UPD = decltype(upd_t)::value, ACC = decltype(acc_t)::value;
  const int fg = lane >> 2, ft = lane & 3;
  // per-pass B operands: W (phase A: b0 = W[16 ks + 2t, + 1][g], b1 = rows + 8) and G (E: b0 =
  // G[2t, 2t + 1][g], b1 = 0), fp16 hi / lo with one power-of-two scale each
  uint32_t wfh[2][2], wfl[2][2], gfh = 0u, gfl = 0u;
  float wsi = 1.f, gsi = 1.f;
  if constexpr (UPD) {
    float wm = 0.f;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int r0 = 16 * ks + 8 * h2 + 2 * ft;
        wm = fmaxf(wm, fmaxf(fabsf(Ws[r0 * 8 + fg]), fabsf(Ws[(r0 + 1) * 8 + fg])));
      }
    const float2 wsc = pow2_scale(warp_max(wm));
    wsi = wsc.y;
#pragma unroll
    for (int ks = 0; ks < 2; ++ks)
#pragma unroll
      for (int h2 = 0; h2 < 2; ++h2) {
        const int r0 = 16 * ks + 8 * h2 + 2 * ft;
        split2(Ws[r0 * 8 + fg], Ws[(r0 + 1) * 8 + fg], wsc.x, wfh[ks][h2], wfl[ks][h2]);
      }
    const float g0 = Gs[(2 * ft) * 8 + fg], g1 = Gs[(2 * ft + 1) * 8 + fg];
    const float2 gsc = pow2_scale(warp_max(fmaxf(fabsf(g0), fabsf(g1))));
    gsi = gsc.y;
    split2(g0, g1, gsc.x, gfh, gfl);
  }
  double paccd[2][4], qaccd[2];
#pragma unroll
  for (int mh = 0; mh < 2; ++mh)
#pragma unroll
    for (int e4 = 0; e4 < 4; ++e4) paccd[mh][e4] = 0.0;
  qaccd[0] = qaccd[1] = 0.0;

  bool parked = false;  // static accumulators parked in pa.park while this warp serves the tail
  for (int64_t j = warp;; j += NWM) {
    if (TG == 0 && j >= J) break;
    const int64_t pos = pbase + j;
    int go = 1;
    if (lane == 0) {
      // static positions are always issued; a tail position is issued unless the pass's total
      // (known once the producer's claims fail) ends before it
      while (ld_acquire_u32(issued) <= (uint32_t)pos) {
        if (j >= J && ld_acquire_u32(&ptot[it & 1]) <= (uint32_t)pos) {
          go = 0;
          break;
        }
        __nanosleep(64);
      }
    }
    if (!__shfl_sync(0xffffffffu, go, 0)) break;
    const uint32_t tg = lane < ns ? *reinterpret_cast<volatile uint32_t*>(tag + lane) : 0xffffffffu;
    const unsigned hit = __ballot_sync(0xffffffffu, (tg >> 1) == (uint32_t)pos && lane < ns);
    const int s = __ffs(hit) - 1;
    const uint32_t ph = __shfl_sync(0xffffffffu, tg, s) & 1u;
    NTT_DCHECK(s >= 0 && s < ns);
    const int64_t tile = TG ? (int64_t)*reinterpret_cast<volatile int32_t*>(tileid + s) : b + j * G;
    const bool tail = j >= J;
    NTT_DCHECK(tile < ntiles && (tail == (tile >= S)));
    const int64_t jt = tile * 128;  // first column of the tile
    if constexpr (ACC) {
      if (tail && !parked) {  // first tail tile of this warp: park the static sums
        double* pk = pa.park + ((size_t)b * NWM + warp) * 320 + lane * 10;
#pragma unroll
        for (int mh = 0; mh < 2; ++mh)
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            pk[mh * 4 + e4] = paccd[mh][e4];
            paccd[mh][e4] = 0.0;
          }
        pk[8] = qaccd[0];
        pk[9] = qaccd[1];
        qaccd[0] = qaccd[1] = 0.0;
        parked = true;
      }
    }
    MBAR_WAIT(&full[s], ph, 2, j);
    unsigned char* st = stages + (size_t)s * SBM;
    unsigned char* hb = st + XBM;
    const uint32_t xs = smem_u32(st);

    // ---- X -> fp16 hi / lo blocks (in place), or the cached blocks' scales
    float xsi[4];
    if (x16_read) {
      const float4 sc4 = *reinterpret_cast<const float4*>(st + XBM + HBM);
      xsi[0] = sc4.x; xsi[1] = sc4.y; xsi[2] = sc4.z; xsi[3] = sc4.w;
    } else {
      unsigned char* gtile = x16_write ? pa.x16 + tile * X16M_STRIDE : nullptr;
#pragma unroll
      for (int bx = 0; bx < 4; ++bx) {
        unsigned char* blk = st + bx * 4096;
        float v[32];
#pragma unroll
        for (int c16 = 0; c16 < 8; ++c16) {
          const float4 f = lds128(blk + lane * 128 + ((c16 ^ (lane & 7)) << 4));
          v[4 * c16] = f.x;
          v[4 * c16 + 1] = f.y;
          v[4 * c16 + 2] = f.z;
          v[4 * c16 + 3] = f.w;
        }
        float m8[8];
#pragma unroll
        for (int q2 = 0; q2 < 8; ++q2)
          m8[q2] = fmaxf(fmaxf(fabsf(v[4 * q2]), fabsf(v[4 * q2 + 1])), fmaxf(fabsf(v[4 * q2 + 2]), fabsf(v[4 * q2 + 3])));
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])), fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        const float2 sc = pow2_scale(warp_max(mx));
        xsi[bx] = sc.y;
        __syncwarp();
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          uint32_t hh[4], ll[4];
#pragma unroll
          for (int p2 = 0; p2 < 4; ++p2) split2(v[8 * k4 + 2 * p2], v[8 * k4 + 2 * p2 + 1], sc.x, hh[p2], ll[p2]);
          *reinterpret_cast<uint4*>(blk + h16_off(lane, k4)) = make_uint4(hh[0], hh[1], hh[2], hh[3]);
          *reinterpret_cast<uint4*>(blk + 2048 + h16_off(lane, k4)) = make_uint4(ll[0], ll[1], ll[2], ll[3]);
          if (gtile) {
            __stcg(reinterpret_cast<uint4*>(gtile + bx * 4096 + h16_off(lane, k4)), make_uint4(hh[0], hh[1], hh[2], hh[3]));
            __stcg(reinterpret_cast<uint4*>(gtile + bx * 4096 + 2048 + h16_off(lane, k4)),
                   make_uint4(ll[0], ll[1], ll[2], ll[3]));
          }
        }
        if (gtile && lane == 0) __stcg(reinterpret_cast<float*>(gtile + XBM) + bx, sc.y);
      }
      __syncwarp();
    }

    // ---- H of this lane's fragment entries: hv[mt][e] = H[2t + (e & 1)][16 mt + g + 8 (e >> 1)]
    float hv[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int e4 = 0; e4 < 4; ++e4)
        hv[mt][e4] = *reinterpret_cast<const float*>(hb + hbox_off(2 * ft + (e4 & 1), 16 * mt + fg + 8 * (e4 >> 1)));
    float hnm = 0.f;  // max |Hn| of the tile (B-operand scale of phase B / Q)
    if constexpr (UPD) {
      float hm = 0.f;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
        hm = fmaxf(hm, fmaxf(fmaxf(fabsf(hv[mt][0]), fabsf(hv[mt][1])), fmaxf(fabsf(hv[mt][2]), fabsf(hv[mt][3]))));
      const float2 hsc = pow2_scale(warp_max(hm));
      const float fE = hsc.y * gsi;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        // E^T rows 16 mt .. + 15 (columns of the tile) = H^T G
        uint32_t ah[4], al[4];
        split2(hv[mt][0], hv[mt][1], hsc.x, ah[0], al[0]);
        split2(hv[mt][2], hv[mt][3], hsc.x, ah[1], al[1]);
        ah[2] = ah[3] = al[2] = al[3] = 0u;  // ranks 8 .. 15: padding
        float de[4] = {0.f, 0.f, 0.f, 0.f};
        mma16816(de, ah, gfh, 0u);
        mma16816(de, ah, gfl, 0u);
        mma16816(de, al, gfh, 0u);
        // S^T rows 16 mt .. + 15 = X^T W over the 32 rows of X (2 k-steps)
        const int bx = mt >> 1, mi = mt & 1;
        float ds[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int mj = lane >> 3;
          const uint32_t off = bx * 4096 + h16_off(16 * ks + (lane & 7) + 8 * (mj >> 1), 2 * mi + (mj & 1));
          uint32_t xh[4], xl[4];
          ldsm_x4_t(xs + off, xh);
          ldsm_x4_t(xs + off + 2048u, xl);
          mma16816(ds, xh, wfh[ks][0], wfh[ks][1]);
          mma16816(ds, xh, wfl[ks][0], wfl[ks][1]);
          mma16816(ds, xl, wfh[ks][0], wfh[ks][1]);
        }
        const float fS = xsi[bx] * wsi;
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) {
          const int k = 2 * ft + (e4 & 1);
          const int64_t col = jt + 16 * mt + fg + 8 * (e4 >> 1);
          float v = mu_q(hv[mt][e4], ds[e4] * fS, de[e4] * fE, eps);
          if (k >= r || col >= n) v = 0.f;  // padded ranks (0/0 when eps = 0), columns beyond n
          else {
            NTT_DCHECK((int64_t)k * n + col < (int64_t)r * n);
            H[(int64_t)k * n + col] = v;
          }
          hv[mt][e4] = v;
          hnm = fmaxf(hnm, fabsf(v));
        }
      }
    } else {
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) hnm = fmaxf(hnm, fabsf(hv[mt][e4]));
    }

    if constexpr (ACC) {
      if constexpr (UPD) {
        // Hn over the stage's H boxes (each entry rewritten by the lane that read it)
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4)
            *reinterpret_cast<float*>(hb + hbox_off(2 * ft + (e4 & 1), 16 * mt + fg + 8 * (e4 >> 1))) = hv[mt][e4];
        __syncwarp();
      }
      const float2 nsc = pow2_scale(warp_max(hnm));
      // B = Hn^T fragments per 16-column k-step: b0 = Hn[g][16 kk + 2t, + 1], b1 = columns + 8
      uint32_t bh[8][2], bl[8][2];
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          const float2 p = *reinterpret_cast<const float2*>(hb + hbox_off(fg, 16 * kk + 8 * h2 + 2 * ft));
          split2(p.x, p.y, nsc.x, bh[kk][h2], bl[kk][h2]);
        }
      // P (32 x 8) += X Hn^T: 2 m-tiles x 8 k-steps (per-block X scale -> one sum per block)
#pragma unroll
      for (int mh = 0; mh < 2; ++mh) {
        float pt[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int bx = 0; bx < 4; ++bx) {
          float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int k2 = 0; k2 < 2; ++k2) {
            const int kk = 2 * bx + k2, mj = lane >> 3;
            const uint32_t off = bx * 4096 + h16_off(16 * mh + (lane & 7) + 8 * (mj & 1), 2 * k2 + (mj >> 1));
            uint32_t xh[4], xl[4];
            ldsm_x4(xs + off, xh);
            ldsm_x4(xs + off + 2048u, xl);
            mma16816(d, xh, bh[kk][0], bh[kk][1]);
            mma16816(d, xh, bl[kk][0], bl[kk][1]);
            mma16816(d, xl, bh[kk][0], bh[kk][1]);
          }
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) pt[e4] = fmaf(d[e4], xsi[bx], pt[e4]);
        }
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) paccd[mh][e4] += (double)(pt[e4] * nsc.y);
      }
      // Q (8 x 8) += Hn Hn^T: A = {b0, 0, b1, 0} (ranks 8 .. 15 padding), B = {b0, b1}
      {
        float dq[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t ah[4] = {bh[kk][0], 0u, bh[kk][1], 0u};
          const uint32_t al[4] = {bl[kk][0], 0u, bl[kk][1], 0u};
          mma16816(dq, ah, bh[kk][0], bh[kk][1]);
          mma16816(dq, ah, bl[kk][0], bl[kk][1]);
          mma16816(dq, al, bh[kk][0], bh[kk][1]);
        }
        qaccd[0] += (double)(dq[0] * (nsc.y * nsc.y));
        qaccd[1] += (double)(dq[1] * (nsc.y * nsc.y));
      }
      // Hn was written over the stage with generic stores: order them before the producer's
      // next TMA (async-proxy) write into this stage
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    } else if (!x16_read) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the in-place X conversion
    }
    __syncwarp();
    if (lane == 0) asm volatile("red.release.cta.shared::cta.or.b32 [%0], %1;" ::"r"(smem_u32(free_mask)), "r"(1u << s) : "memory");
    if constexpr (ACC) {
      const int64_t ut = tile - S;  // tail: group ut / kTailGroup, member ut % kTailGroup
      if (tail && (ut % kTailGroup) >= kTailGroup - NWM) {
        // this warp's last tile of the group (members u, u + 8, ...): their sums -> slot G + 8 g + u % 8
        const int mr = m * r;
        double* dst = pa.part + ((int64_t)G + NWM * (ut / kTailGroup) + (ut % NWM)) * (mr + r * r);
#pragma unroll
        for (int mh = 0; mh < 2; ++mh)
#pragma unroll
          for (int e4 = 0; e4 < 4; ++e4) {
            const int row = 16 * mh + fg + 8 * (e4 >> 1), k = 2 * ft + (e4 & 1);
            if (row < m && k < r) dst[row * r + k] = paccd[mh][e4];
            paccd[mh][e4] = 0.0;
          }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          if (fg < r && 2 * ft + q < r) dst[mr + fg * r + 2 * ft + q] = qaccd[q];
          qaccd[q] = 0.0;
        }
      }
    }
  }

  if constexpr (ACC) {
    if (parked) {  // the static sums back (the tail's were flushed to their slots)
      const double* pk = pa.park + ((size_t)b * NWM + warp) * 320 + lane * 10;
#pragma unroll
      for (int mh = 0; mh < 2; ++mh)
#pragma unroll
        for (int e4 = 0; e4 < 4; ++e4) paccd[mh][e4] = pk[mh * 4 + e4];
      qaccd[0] = pk[8];
      qaccd[1] = pk[9];
    }
    // ---- fixed-order CTA reduction of the warps' fp64 partials: red[w][0 .. 256) = P (32 x 8),
    // red[w][256 .. 320) = Q (8 x 8)
    asm volatile("bar.sync 1, %0;" ::"r"(NWM * 32) : "memory");
    double* red = reinterpret_cast<double*>(stages);
#pragma unroll
    for (int mh = 0; mh < 2; ++mh)
#pragma unroll
      for (int e4 = 0; e4 < 4; ++e4)
        red[warp * 320 + (16 * mh + fg + 8 * (e4 >> 1)) * 8 + 2 * ft + (e4 & 1)] = paccd[mh][e4];
    red[warp * 320 + 256 + fg * 8 + 2 * ft] = qaccd[0];
    red[warp * 320 + 256 + fg * 8 + 2 * ft + 1] = qaccd[1];
    asm volatile("bar.sync 1, %0;" ::"r"(NWM * 32) : "memory");
    const int mr = m * r, rr = r * r;
    double* Pb = persist ? pa.part + b * (mr + rr) : Ppart + b * mr;
    double* Qb = persist ? pa.part + b * (mr + rr) + mr : Qpart + b * rr;
    for (int e = tid; e < 320; e += NWM * 32) {
      const bool isQ = e >= 256;
      const int row = isQ ? (e - 256) >> 3 : e >> 3, k = e & 7;
      if (k >= r || (isQ ? row >= r : row >= m)) continue;
      double sum = 0.0;
      for (int w = 0; w < NWM; ++w) sum += red[w * 320 + e];
      if (isQ) Qb[row * r + k] = sum;
      else Pb[row * r + k] = sum;
    }
  }
  };  // pass_tiles
  using T_ = std::true_type;
  using F_ = std::false_type;
  if (!do_update) pass_tiles(F_{}, T_{});
  else if (do_acc) pass_tiles(T_{}, T_{});
  else pass_tiles(T_{}, F_{});
  }  // consumer warps
  if (!persist || !do_acc) break;
  persist_step<8>(pa, epoch, m, r, eps, Ws, Gs, reinterpret_cast<double*>(stages), it, xs0);
  }  // passes
  if (persist) xseq_store(pa, xs0);
}

size_t fixed_bytes_m() { return 32 * 8 * 4 + 256 + 2 * 24 * 8 + 256 + 1024; }

int stages_m() {
  int ns = (int)((SMEM_BUDGET - fixed_bytes_m()) / SBM);
  return ns > 24 ? 24 : ns;
}

cudaError_t launch_m(const CUtensorMap& mx, const CUtensorMap& mh, int m, int64_t n, int r, const float* W,
                     const double* Gpart, int nG, float eps, float* H, double* Ppart, double* Qpart, int mode, int grid,
                     int evict_first, const PersistArgs& pa, cudaStream_t st) {
  const int ns = stages_m();
  const size_t smem = (size_t)ns * SBM + fixed_bytes_m();
  if (pa.iters > 0 && persist_scratch_bytes(m, r, 8, (NWM + 1) * 32) > (size_t)ns * SBM) return cudaErrorInvalidConfiguration;
  cudaError_t e = smem_optin((const void*)(k_fused_m), smem);
  if (e != cudaSuccess) return e;
  return launch_maybe_coop(k_fused_m, grid, (NWM + 1) * 32, smem, st, pa.iters > 0, mx, mh, m, n, r, W, Gpart, nG,
                           eps, H, Ppart, Qpart, mode, ns, evict_first, pa);
}

// ------------------------------------------------------------ W update v2 --
// CTA c owns rows [c*RB, c*RB+RB) with RB*r <= 64 entries; 1024 threads = 64
// entries x 16 chunks of partials; each thread sums its chunk with 4
// independent accumulators (latency hiding), chunks are combined in order --
// a fixed summation tree, so results are deterministic.
constexpr int WU2_CH = 16;

__device__ __forceinline__ double chunk_sum(const double* __restrict__ base, int64_t stride, int b0, int b1) {
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int bq = b0;
  for (; bq + 3 < b1; bq += 4) {
    s0 += base[(int64_t)bq * stride];
    s1 += base[(int64_t)(bq + 1) * stride];
    s2 += base[(int64_t)(bq + 2) * stride];
    s3 += base[(int64_t)(bq + 3) * stride];
  }
  for (; bq < b1; ++bq) s0 += base[(int64_t)bq * stride];
  return (s0 + s1) + (s2 + s3);
}

template <int R>
__global__ void __launch_bounds__(64 * WU2_CH)
k_wupdate2(float* __restrict__ W, int64_t m, int r, const double* __restrict__ Ppart, int nP,
           const double* __restrict__ Qpart, int nQ, float eps, double* __restrict__ Gpart) {
  constexpr int RB = (64 / R) > 0 ? (64 / R) : 1;
  __shared__ double part[WU2_CH][64];
  __shared__ double Qs[R * R];
  __shared__ double Ps[RB * R];
  __shared__ float Wn[RB][R];
  const int t = threadIdx.x, e = t & 63, c = t >> 6;
  const int rr = r * r;
  // Q = sum of partials
  for (int q0 = 0; q0 < rr; q0 += 64) {
    const int qe = q0 + e;
    double sum = 0.0;
    if (qe < rr) {
      const int b0 = (int)((int64_t)nQ * c / WU2_CH), b1 = (int)((int64_t)nQ * (c + 1) / WU2_CH);
      sum = chunk_sum(Qpart + qe, rr, b0, b1);
    }
    part[c][e] = sum;
    __syncthreads();
    if (c == 0 && qe < rr) {
      double tot = 0.0;
#pragma unroll
      for (int cc = 0; cc < WU2_CH; ++cc) tot += part[cc][e];
      Qs[(qe / r) * R + (qe % r)] = tot;
    }
    __syncthreads();
  }
  // P rows of this CTA
  const int64_t i0 = (int64_t)blockIdx.x * RB;
  const int rows = (int)min((int64_t)RB, m - i0);
  const int64_t mr = m * r;
  {
    double sum = 0.0;
    const bool ok = e < rows * r;
    if (ok) {
      const int b0 = (int)((int64_t)nP * c / WU2_CH), b1 = (int)((int64_t)nP * (c + 1) / WU2_CH);
      sum = chunk_sum(Ppart + i0 * r + e, mr, b0, b1);
    }
    part[c][e] = sum;
    __syncthreads();
    if (c == 0 && ok) {
      double tot = 0.0;
#pragma unroll
      for (int cc = 0; cc < WU2_CH; ++cc) tot += part[cc][e];
      Ps[(e / r) * R + (e % r)] = tot;
    }
    __syncthreads();
  }
  if (t < RB) {
    if (t < rows) {
      const int64_t i = i0 + t;
      double w[R];
#pragma unroll
      for (int k = 0; k < R; ++k) w[k] = (k < r) ? (double)W[i * r + k] : 0.0;
#pragma unroll
      for (int k = 0; k < R; ++k) {
        if (k >= r) {
          Wn[t][k] = 0.0f;
          continue;
        }
        double dd = 0.0;
#pragma unroll
        for (int l = 0; l < R; ++l)
          if (l < r) dd += w[l] * Qs[l * R + k];
        Wn[t][k] = (float)mu_quot(w[k], Ps[t * R + k], dd, (double)eps);
      }
      for (int k = 0; k < r; ++k) W[i * r + k] = Wn[t][k];
    } else {
#pragma unroll
      for (int k = 0; k < R; ++k) Wn[t][k] = 0.0f;
    }
  }
  __syncthreads();
  for (int qq = t; qq < rr; qq += 64 * WU2_CH) {
    const int k = qq / r, l = qq % r;
    double sum = 0.0;
    for (int ii = 0; ii < RB; ++ii) sum += (double)Wn[ii][k] * (double)Wn[ii][l];
    Gpart[(int64_t)blockIdx.x * rr + qq] = sum;
  }
}

int rb2_for(int r) {
  int R = r <= 2 ? 2 : r <= 4 ? 4 : r <= 8 ? 8 : r <= 16 ? 16 : r <= 32 ? 32 : 64;
  return (64 / R) > 0 ? 64 / R : 1;
}

}  // namespace

bool fused_supported(int64_t m, int64_t n, int r, int64_t ldx, const void* X, const void* H) {
  // ranks up to 8 (k_fused, m <= 40) or 16 (k_fused_c's RK = 16 class, 40 < m <= 256)
  if (m < 1 || m > 256 || r < 1 || r > (m > 40 ? 16 : 8) || n < 4) return false;
  if ((n & 3) || (ldx & 3)) return false;
  if ((reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(H) & 15)) return false;
  if (n > (int64_t)INT32_MAX - 256) return false;
  return true;
}

int fused_partials(int64_t m, int64_t n, int r, int num_sms) {
  const int g = fused_grid(m, n, r, num_sms);
  return g;
}

int fused_grid(int64_t m, int64_t n, int r, int num_sms) {
  (void)r;
  if (m <= 40) {
    int64_t ntiles = (n + BN - 1) / BN;
    return (int)(ntiles < num_sms ? ntiles : num_sms);
  }
  int64_t ntiles = (n + BNC - 1) / BNC;
  // k_fused_c: two CTAs of 4 consumer warps per SM; one CTA of 8 for the RK = 16 class at MP = 256
  const int cps = (m > 128 && r > 8) ? 1 : 2;
  return (int)(ntiles < cps * num_sms ? ntiles : cps * num_sms);
}

size_t fused_scratch_bytes(int64_t, int64_t, int, int) { return 0; }

// the tensor-core one-pass kernel for 16 < m <= 32 (k_fused_m) takes the shape (MU only)
bool fused_m_ok(int64_t m, int64_t n, int r) { return m > 16 && m <= 32 && r <= 8 && (n % 32) == 0; }

// Dynamic tail of the persistent k_fused_m (PersistArgs::tail_groups): ~kTailPerCta tiles per CTA
// at the end of every pass, in groups of kTailGroup, when each CTA has > 2 kTailPerCta tiles.  Measured:
// CTA pass times spread 4-7 % (systematic by SM group), i.e. 35-40 us of barrier wait per pass on
// config 3 step 1.  NTT_NO_TAIL=1: static schedule.
int fused_tail_groups(int64_t m, int64_t n, int r, int grid) {
  constexpr int64_t kTailPerCta = 40;
  const bool off = getenv("NTT_NO_TAIL") != nullptr;
  if (off || !fused_m_ok(m, n, r) || grid < 1) return 0;
  const int64_t ntiles = (n + 127) / 128, jfull = ntiles / grid;
  if (jfull <= 2 * kTailPerCta) return 0;
  return (int)((ntiles - (jfull - kTailPerCta) * grid) / kTailGroup);
}

size_t fused_x16_bytes(int64_t m, int64_t n) {
  if (m > 16 && m <= 32 && (n % 32) == 0) return (size_t)((n + 127) / 128) * (size_t)X16M_STRIDE;
  if (m <= 40) return 0;
  return (size_t)((n + BNC - 1) / BNC) * (size_t)(((m + 31) / 32) * 4096 + 128);
}
void fused_destroy(FusedCtx&) {}

struct FusedPlan {
  bool x3d;  // X (and staged H) through 3-D maps: one box per 128-column tile
  bool hd;   // lanes load H directly (no H boxes in the stage)
  int bn;    // tile width (columns)
};

// the k_fused variant launch_fused picks for m <= 40
FusedPlan fused_plan(int64_t m, int64_t n, int r) {
  const int ux = ux_for(m);
  FusedPlan p;
  // X (and staged H) through 3-D maps {32 cols, 8 rows, n / 32 blocks}: one 4 KB box per
  // 128-column tile instead of four 1 KB boxes (TMA wants multi-KB transactions, tools/tmabench.cu)
  p.x3d = (n % 32) == 0;
  // with the 3-D maps staging H through TMA (one 4 KB box per tile) beats the lanes' direct
  // loads, which cannot keep enough bytes in flight (tools/membench.cu): config 4 step 1
  // 59.4 -> 53.7 ms, steps 2-5 -2 to -5 %; without them direct H loads win where H is a large
  // share of the traffic (m <= 16 or r < 8)
  p.hd = p.x3d ? false : (ux <= 2 || r < 8);
  p.bn = 128;
  return p;
}

bool fused_fold_ok(int64_t m, int64_t n, int r, int64_t ldx, const void* X, const void* H0, const void* H1) {
  if (m > 40 || !fused_supported(m, n, r, ldx, X, H0) || !fused_supported(m, n, r, ldx, X, H1)) return false;
  if ((reinterpret_cast<uintptr_t>(H0) & 15) || (reinterpret_cast<uintptr_t>(H1) & 15) || (n & 3)) return false;
  const FusedPlan p = fused_plan(m, n, r);
  return !p.hd && p.bn == 128;
}

cudaError_t launch_fused(const float* X, int64_t ldx, int64_t m, int64_t n, int r, const float* W, const double* Gpart,
                         int nG, float eps, float* H, double* Ppart, double* Qpart, int mode, int grid,
                         cudaStream_t st, const PersistArgs* pap) {
  const PersistArgs pa = pap ? *pap : PersistArgs{0, nullptr, nullptr, nullptr, nullptr, nullptr};
  const int evict_first = ((double)m * (double)n * 4.0 > 48e6) ? 1 : 0;
  if (m > 40) {
    const int MPc = m <= 128 ? 128 : 256;
    CUtensorMap mx, mh;
    cudaError_t e = make_map(&mx, X, (uint64_t)n, (uint64_t)m, (uint64_t)ldx, (uint32_t)MPc);
    if (e != cudaSuccess) return e;
    const int RKc = r <= 8 ? 8 : 16;
    e = make_map(&mh, H, (uint64_t)n, (uint64_t)r, (uint64_t)n, (uint32_t)RKc);
    if (e != cudaSuccess) return e;
#define LC(MP_, RK_) \
  return launch_c<MP_, 4, RK_>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, evict_first, pa, st)
    if (MPc == 128) {
      if (RKc == 8) LC(128, 8);
      LC(128, 16);
    }
    if (RKc == 8) LC(256, 8);
#undef LC
    return launch_c<256, 8, 16>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, evict_first, pa, st);
#undef LC
  }
  if (!pa.bcdL && fused_m_ok(m, n, r)) {  // MU on tensor cores (k_fused_m)
    CUtensorMap mx, mh;
    cudaError_t e = make_map3(&mx, X, (uint64_t)n, (uint64_t)m, (uint64_t)ldx, 32u, 4u);
    if (e != cudaSuccess) return e;
    if ((e = make_map3(&mh, H, (uint64_t)n, (uint64_t)r, (uint64_t)n, 8u, 4u)) != cudaSuccess) return e;
    return launch_m(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, evict_first, pa, st);
  }
  const int ux = ux_for(m);
  CUtensorMap mx, mh, mb0, mb1;
  const FusedPlan fp = fused_plan(m, n, r);
  int ef = evict_first;
  cudaError_t e;
  if (fp.x3d) {  // one 3-D box per 128-column tile
    e = make_map3(&mx, X, (uint64_t)n, (uint64_t)m, (uint64_t)ldx, (uint32_t)(ux * 8), 4u);
    ef |= 2;
  } else {
    e = make_map(&mx, X, (uint64_t)n, (uint64_t)m, (uint64_t)ldx, (uint32_t)(ux * 8));
  }
  if (e != cudaSuccess) return e;
  const int rc = rcls_for(r);
  const bool hd = fp.hd;
  // H boxes (staged path): 3-D as well when X uses the 3-D map (block stride 128 B of row pitch n)
  auto hmap = [&](CUtensorMap* mp, const float* base) {
    return (ef & 2) && !hd && (n % 32) == 0 ? make_map3(mp, base, (uint64_t)n, (uint64_t)r, (uint64_t)n, 8u, 4u)
                                            : make_map(mp, base, (uint64_t)n, (uint64_t)r, (uint64_t)n, 8u);
  };
  e = hmap(&mh, H);
  if (e != cudaSuccess) return e;
  if (pa.bcdFold) {  // BCD H_m fold: both H buffers (fused_fold_ok() said this variant runs)
    if (hd || !pa.Hout || !pa.Hout2 || !pa.bcdRole) return cudaErrorNotSupported;
    if ((e = hmap(&mb0, pa.Hout)) != cudaSuccess) return e;
    if ((e = hmap(&mb1, pa.Hout2)) != cudaSuccess) return e;
#define LFF(RR, UU) \
  return launch_t<RR, UU, 8, false, 128, true>(mx, mb0, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, ef, pa, st, &mb1)
    if (rc == 2) {
      if (ux == 1) LFF(2, 1);
      if (ux == 2) LFF(2, 2);
      if (ux == 4) LFF(2, 4);
      LFF(2, 5);
    }
    if (rc == 6) {
      if (ux == 1) LFF(6, 1);
      if (ux == 2) LFF(6, 2);
      if (ux == 4) LFF(6, 4);
      LFF(6, 5);
    }
    if (rc == 4) {
      if (ux == 1) LFF(4, 1);
      if (ux == 2) LFF(4, 2);
      if (ux == 4) LFF(4, 4);
      LFF(4, 5);
    }
    if (ux == 1) LFF(8, 1);
    if (ux == 2) LFF(8, 2);
    if (ux == 4) LFF(8, 4);
    LFF(8, 5);
#undef LFF
  }
#define LF(RR, UU)                                                                                                   \
  return hd ? launch_t<RR, UU, 8, true, 128>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, ef, pa, st) \
            : launch_t<RR, UU, 8, false, 128>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, ef, pa, st)
  if (rc == 2) {
    if (ux == 1) LF(2, 1);
    if (ux == 2) LF(2, 2);
    if (ux == 4) LF(2, 4);
    LF(2, 5);
  }
  if (rc == 6) {  // r = 5, 6 (config 4): less padded work than the R = 8 class
    if (ux == 1) LF(6, 1);
    if (ux == 2) LF(6, 2);
    if (ux == 4) LF(6, 4);
    LF(6, 5);
  }
  if (rc == 4) {
    if (ux == 1) LF(4, 1);
    if (ux == 2) LF(4, 2);
    if (ux == 4) LF(4, 4);
    LF(4, 5);
  }
  if (ux == 1) LF(8, 1);
  if (ux == 2) LF(8, 2);
  if (ux == 4) LF(8, 4);
  LF(8, 5);
#undef LF
}

int wupdate2_ctas(int64_t m, int r) {
  const int rb = rb2_for(r);
  return (int)((m + rb - 1) / rb);
}

cudaError_t launch_wupdate2(float* W, int64_t m, int r, const double* Ppart, int nP, const double* Qpart, int nQ,
                            float eps, double* Gpart, cudaStream_t st) {
  const int grid = wupdate2_ctas(m, r);
#define WU(RR) k_wupdate2<RR><<<grid, 64 * WU2_CH, 0, st>>>(W, m, r, Ppart, nP, Qpart, nQ, eps, Gpart)
  if (r <= 2) WU(2);
  else if (r <= 4) WU(4);
  else if (r <= 8) WU(8);
  else if (r <= 16) WU(16);
  else if (r <= 32) WU(32);
  else WU(64);
#undef WU
  return cudaGetLastError();
}

}  // namespace ntt
