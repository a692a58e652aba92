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
#include <cstdio>
#include <cstdlib>
#include <utility>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "mu_fused.h"

namespace ntt {

namespace {

constexpr int NW = 8;               // consumer warps
constexpr int NT = (NW + 1) * 32;   // + 1 TMA producer warp
constexpr int BN = 128;             // tile columns
constexpr int HN_FLOATS = 1168;     // per-warp transposed Hn tile (padded)
constexpr int SMEM_BUDGET = 232448; // 227 KB opt-in

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// try_wait in a C++ loop (not an asm-internal branch loop): the compiler must
// see the divergent spin to place reconvergence before warp-synchronous code.
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try(bar, parity)) {
  }
}
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
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// one 3-D box {32 cols, rows, blocks} = `blocks` consecutive 32-column boxes in one transaction
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
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

// Reduce the per-CTA partials and apply the W update in every CTA (see above).
// Ws: [i * 8 + k] (rows >= m stay zero), Gs: [k * 8 + l]; scr: >= (L + 16) doubles + m*8 floats
// + 256 doubles of smem.  Global reads are issued in independent batches (L2 latency is ~1 us).
// W layout in smem: row-major [i * 8 + k], or (pairs) [i/2][k/2][i%2][k%2] so that a
// lane reading ranks (2g, 2g+1) of rows (i, i+1) issues one 128-bit load (k_fused_c)
__device__ __forceinline__ int widx(int i, int k, bool pairs) {
  return pairs ? ((i >> 1) << 4) + ((k >> 1) << 2) + ((i & 1) << 1) + (k & 1) : (i << 3) + k;
}

__device__ void persist_step(const PersistArgs& pa, unsigned& epoch, int m, int r, float eps, float* Ws, float* Gs,
                             double* scr, int it, bool pairs = false) {
  const int L = m * r + r * r;
  const int T = blockDim.x, tid = threadIdx.x;
  pstamp(pa, it, 1);
  if (gridDim.x > 1) {
    grid_sync(pa.ctr, epoch);
    pstamp(pa, it, 2);
    const int G = gridDim.x;
    const int SL = (L + G - 1) / G;
    const int e0 = blockIdx.x * SL;
    const int ne = min(L, e0 + SL) - e0;
    if (ne > 0) {
      int C = T / ne;
      C = C < 1 ? 1 : (C > 32 ? 32 : C);
      for (int t = tid; t < ne * C; t += T) {
        const int e = t % ne, c = t / ne;
        const int g0 = (int)((int64_t)G * c / C), g1 = (int)((int64_t)G * (c + 1) / C);
        const double* src = pa.part + e0 + e;
        double a[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) a[q] = 0.0;
        for (int g = g0; g < g1; g += 8) {
#pragma unroll
          for (int q = 0; q < 8; ++q)
            if (g + q < g1) a[q] += __ldcg(src + (int64_t)(g + q) * L);
        }
        scr[c * ne + e] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
      }
      __syncthreads();
      for (int e = tid; e < ne; e += T) {
        double sv = 0.0;
        for (int c = 0; c < C; ++c) sv += scr[c * ne + e];
        __stcg(pa.red + e0 + e, sv);
      }
    }
    grid_sync(pa.ctr, epoch);
  } else {
    __syncthreads();  // single CTA: its own partial is the sum
  }
  pstamp(pa, it, 3);
  const double* srcv = gridDim.x > 1 ? pa.red : pa.part;
  for (int e0 = 0; e0 < L; e0 += 8 * T) {
    double v[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q * T + tid;
      v[q] = e < L ? __ldcg(srcv + e) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int e = e0 + q * T + tid;
      if (e < L) scr[e] = v[q];
    }
  }
  __syncthreads();
  double* P = scr;           // m x r
  double* Q = scr + m * r;   // r x r
  float* Wn = reinterpret_cast<float*>(scr + L + 16);
  double* Gp = scr + L + 16 + (m * 8 + 1) / 2 + 8;  // [C][64] Gram chunk partials
  for (int e = tid; e < m * 8; e += T) {
    const int i = e >> 3, k = e & 7;
    float v = 0.0f;
    if (k < r) {
      double d = 0.0;
      for (int l = 0; l < r; ++l) d += (double)Ws[widx(i, l, pairs)] * Q[l * r + k];
      v = (float)mu_quot((double)Ws[widx(i, k, pairs)], P[i * r + k], d, (double)eps);
    }
    Wn[e] = v;
  }
  __syncthreads();
  for (int e = tid; e < m * 8; e += T) Ws[widx(e >> 3, e & 7, pairs)] = Wn[e];
  // G = Wn^T Wn: 64 entries x C row chunks (fixed order), then combine
  const int GC = T / 64 < 1 ? 1 : (T / 64 > 4 ? 4 : T / 64);
  for (int t = tid; t < 64 * GC; t += T) {
    const int e = t & 63, c = t >> 6;
    const int k = e >> 3, l = e & 7;
    const int i0 = m * c / GC, i1 = m * (c + 1) / GC;
    double s0 = 0.0, s1 = 0.0;
    if (k < r && l < r) {
      int i = i0;
      for (; i + 1 < i1; i += 2) {
        s0 += (double)Wn[i * 8 + k] * (double)Wn[i * 8 + l];
        s1 += (double)Wn[(i + 1) * 8 + k] * (double)Wn[(i + 1) * 8 + l];
      }
      if (i < i1) s0 += (double)Wn[i * 8 + k] * (double)Wn[i * 8 + l];
    }
    Gp[c * 64 + e] = s0 + s1;
  }
  __syncthreads();
  for (int e = tid; e < 64; e += T) {
    double sg = 0.0;
    for (int c = 0; c < GC; ++c) sg += Gp[c * 64 + e];
    Gs[e] = (float)sg;
  }
  if (blockIdx.x == 0)
    for (int e = tid; e < m * r; e += T) pa.Wout[e] = Wn[(e / r) * 8 + (e % r)];
  __syncthreads();
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
  persist_step(pa, epoch, m, r, eps, Ws, Gs, reinterpret_cast<double*>(stages), it);
  }  // passes
}


// ===========================================================================
// Variant C: CTA-cooperative tiles for 40 < m <= 256 (rank padded to 8).
// Small CTAs (4 consumer warps + 1 TMA warp, <= 112 KB smem) so TWO CTAs share
// an SM and one CTA's serial sections (S reduction, H update, barriers) overlap
// the other's FMA phases.  Tile = 32 columns x MP rows (one SWIZZLE_128B box)
// + the 8 x 32 H box.  Phase A splits the m-long dot products across the 4
// warps (warp w owns rows [RW w, RW w + RW)), reduces the partial S tiles
// through smem in fixed order; 128 threads form E = G H and Hn (2 entries
// each).  Phase B: warp w owns the same rows of P = X Hn^T in sub-chunks of 32
// (lanes = row block x 8-column slice, reduce-scatter over the slices, fp64
// accumulation), and rows 2w, 2w+1 of Q = Hn Hn^T.  Rows are disjoint across
// warps, so per-CTA partials need no cross-warp reduction.
// ===========================================================================
constexpr int BNC = 32;
constexpr int NWC = 4;                  // consumer warps per CTA
constexpr int NTC = (NWC + 1) * 32;
constexpr int HNC_FLOATS = 32 * 8 + 16; // transposed Hn tile [c][k] + 4 floats per 8-column group
constexpr int SMEM_C = 113 * 1024;      // two CTAs per SM

__device__ __forceinline__ int hnc_idx(int c, int k) { return c * 8 + k + 4 * (c >> 3); }

template <int MP, int NW>
__global__ void __launch_bounds__((NW + 1) * 32, NW == 4 ? 2 : 1)
k_fused_c(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmH, int m, int64_t n, int r,
          const float* __restrict__ W, const double* __restrict__ Gpart, int nG, float eps, float* __restrict__ H,
          double* __restrict__ Ppart, double* __restrict__ Qpart, int mode, int ns, int evict_first,
          PersistArgs pa) {
  extern __shared__ unsigned char smem_raw[];
  // keep the shared address space visible to the compiler (LDS/STS, not generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int RW = MP / NW;           // rows per warp (32 or 64)
  constexpr int NCH = RW / 32;          // phase-B sub-chunks of 32 rows
  static_assert(RW >= 32 && RW % 32 == 0, "k_fused_c: at least 32 rows per consumer warp");
  constexpr int HH = 256 / (NW * 32);   // H-update (k, c) pairs per thread
  constexpr int QR = 8 / NW;            // Q rows per warp
  constexpr bool WREG = (RW == 32);     // W rows of this warp kept in registers
  constexpr int NTHR = (NW + 1) * 32;
  constexpr uint32_t XB = MP * 128u;
  constexpr uint32_t SB = XB + 1024u;
  unsigned char* stages = smem;
  float* Sred = reinterpret_cast<float*>(smem + (size_t)ns * SB);  // [NW][8 k][32 c]
  float* Gs = Sred + NW * 8 * 32;                                    // 8 x 8
  float* Hn = Gs + 64;                                               // HNC_FLOATS
  float* Wc = Hn + HNC_FLOATS;                                       // MP x 8 (rank padded)
  uint64_t* full = reinterpret_cast<uint64_t*>(Wc + MP * 8);
  uint64_t* empty = full + ns;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool persist = pa.iters > 0;
  // BCD mode (PersistArgs::bcdL; see k_fused): row scales of H_m (smem), 1 / L_H, output buffer
  const bool bcd = pa.bcdL != nullptr;
  __shared__ float bsh[8];
  if (tid < 8) bsh[tid] = (bcd && tid < r) ? (float)pa.bcdS[tid] : 1.f;
  const float binvL = (bcd && *pa.bcdL > 0.0) ? (float)(1.0 / *pa.bcdL) : 0.f;
  float* const Ho = (bcd && pa.Hout) ? ((pa.bcdRole && *pa.bcdRole != 0.0) ? pa.Hout2 : pa.Hout) : H;
  if (!persist && (mode & kFusedUpdate)) {
    const int rr = r * r;
    for (int e = tid; e < 64; e += NTHR) {
      int k = e >> 3, l = e & 7;
      double sum = 0.0;
      if (k < r && l < r)
        for (int bq = 0; bq < nG; ++bq) sum += Gpart[(int64_t)bq * rr + k * r + l];
      Gs[e] = (float)sum;
    }
  }
#ifdef NTT_FC_PAIR_A
  constexpr bool COLA = false;
#else
  // phase A with lanes = (2 columns, 4 ranks): X by LDS.64 (one 128-byte row per warp) and W
  // by one half-warp-uniform LDS.128 per row; the (4 columns x 2 ranks) lane layout read X by
  // 128-bit loads that 4 lanes share (4 wavefronts per row, tools/ldsbench.cu), and the
  // (1 column x 8 ranks) layout spent 2 x 2 wavefronts per row on uniform LDS.128s of W
  constexpr bool COLA = !WREG;
#endif
  constexpr bool WPAIR = !WREG && !COLA;  // W in row-pair layout (one 128-bit load per 2 rows in phase A)
  for (int e = tid; e < MP * 8; e += NTHR) {
    const int i = e >> 3, k = e & 7;
    Wc[widx(i, k, WPAIR)] = (i < m && k < r) ? W[(int64_t)i * r + k] : 0.0f;
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
  const int64_t J = (ntiles > b) ? (ntiles - b + gridDim.x - 1) / gridDim.x : 0;

  unsigned epoch = 0;
  int ring_s = 0;          // ring stage / parity of the next tile (continues across passes;
  uint32_t ring_ph = 0;    // incremental: a 64-bit pos % ns was a division call per tile)
  const int nit = persist ? pa.iters + 1 : 1;
  for (int it = 0; it < nit; ++it) {
  const int md = persist ? (it == 0 ? kFusedAcc : (kFusedUpdate | (it < pa.iters ? kFusedAcc : 0))) : mode;
  const bool do_update = (md & kFusedUpdate) != 0;
  const bool do_acc = (md & kFusedAcc) != 0;
  const int64_t pbase = (int64_t)it * J;
  pstamp(pa, it, 0);
  if (warp == NW) {
    if (lane == 0) {
      uint64_t policy;
      if (evict_first)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
      for (int64_t j = 0; j < J; ++j) {
        const int s = ring_s;
        const uint32_t ph = ring_ph;
        if (++ring_s == ns) {
          ring_s = 0;
          ring_ph ^= 1u;
        }
        MBAR_WAIT(&empty[s], ph ^ 1u, 3, j);
        mbar_expect_tx(&full[s], SB);
        const int col0 = (int)((b + j * gridDim.x) * BNC);
        unsigned char* st = stages + (size_t)s * SB;
        tma_load_2d(st, &tmX, col0, 0, &full[s], policy);
        tma_load_2d(st + XB, &tmH, col0, 0, &full[s], policy);
      }
    }
  } else {

  const int q = lane & 7, g = lane >> 3;   // phase A: columns 4q..4q+3, ranks 2g, 2g+1
  const int rb = lane & 7, cs = lane >> 3; // phase B: rows rb + 8u of a 32-row chunk, columns 8cs..8cs+7
  double accd[NCH][8];
#pragma unroll
  for (int h = 0; h < NCH; ++h)
#pragma unroll
    for (int v = 0; v < 8; ++v) accd[h][v] = 0.0;
  double qd[QR];
#pragma unroll
  for (int qq = 0; qq < QR; ++qq) qd[qq] = 0.0;
  const bool h1 = (lane >> 4) & 1, h0 = (lane >> 3) & 1;
  constexpr int NBAR = NW * 32;
  // this warp's W rows (ranks 2g, 2g+1) in registers when it owns 32 rows
  float2 wreg[WREG ? 32 : 1];
  if constexpr (WREG) {
#pragma unroll
    for (int v = 0; v < 32; ++v) wreg[v] = *reinterpret_cast<const float2*>(Wc + widx(warp * RW + v, 2 * g, false));
  }

  for (int64_t j = 0; j < J; ++j) {
    const int s = ring_s;
    const uint32_t ph = ring_ph;
    if (++ring_s == ns) {
      ring_s = 0;
      ring_ph ^= 1u;
    }
    MBAR_WAIT(&full[s], ph, 4, j);
    const unsigned char* st = stages + (size_t)s * SB;
    const int64_t jt = (b + j * gridDim.x) * BNC;

    if (do_update) {
      // ---- phase A: partial S over this warp's rows
      float2 sa = f2(0.f, 0.f), sb = f2(0.f, 0.f), sc = f2(0.f, 0.f), sd = f2(0.f, 0.f);
      if constexpr (COLA) {
        // lane = (cp = lane & 15: columns 2cp, 2cp+1; kh = lane >> 4: ranks 4kh..4kh+3);
        // sa..sd = S[4kh + 0..3][2cp..2cp+1]
        const int cp = lane & 15, kh = lane >> 4;
        const unsigned char* xb = st + (size_t)(warp * RW) * 128 + (cp & 1) * 8;
        const float* wb = Wc + warp * RW * 8 + 4 * kh;
#pragma unroll 8
        for (int v = 0; v < RW; ++v) {
          const float2 x = *reinterpret_cast<const float2*>(xb + v * 128 + (((cp >> 1) ^ (v & 7)) << 4));
          const float4 w = *reinterpret_cast<const float4*>(wb + v * 8);
          sa = __ffma2_rn(bc(w.x), x, sa);
          sb = __ffma2_rn(bc(w.y), x, sb);
          sc = __ffma2_rn(bc(w.z), x, sc);
          sd = __ffma2_rn(bc(w.w), x, sd);
        }
        float* sr = Sred + (warp * 8 + 4 * kh) * 32 + 2 * cp;
        *reinterpret_cast<float2*>(sr) = sa;
        *reinterpret_cast<float2*>(sr + 32) = sb;
        *reinterpret_cast<float2*>(sr + 64) = sc;
        *reinterpret_cast<float2*>(sr + 96) = sd;
      } else if constexpr (WREG) {
#pragma unroll
        for (int v = 0; v < RW; ++v) {
          const int i = warp * RW + v;
          const float4 x = lds128(st + i * 128 + ((q ^ (i & 7)) << 4));
          const float2 x01 = f2(x.x, x.y), x23 = f2(x.z, x.w);
          const float2 wv = wreg[v & 31];
          sa = __ffma2_rn(bc(wv.x), x01, sa);
          sb = __ffma2_rn(bc(wv.x), x23, sb);
          sc = __ffma2_rn(bc(wv.y), x01, sc);
          sd = __ffma2_rn(bc(wv.y), x23, sd);
        }
      } else {
#pragma unroll 4
        for (int v = 0; v < RW; v += 2) {
          const int i = warp * RW + v;
          const float4 xa = lds128(st + i * 128 + ((q ^ (i & 7)) << 4));
          const float4 xb = lds128(st + (i + 1) * 128 + ((q ^ ((i + 1) & 7)) << 4));
          // W[i][2g], W[i][2g+1], W[i+1][2g], W[i+1][2g+1]
          const float4 w4 = *reinterpret_cast<const float4*>(Wc + widx(i, 2 * g, true));
          sa = __ffma2_rn(bc(w4.x), f2(xa.x, xa.y), sa);
          sb = __ffma2_rn(bc(w4.x), f2(xa.z, xa.w), sb);
          sc = __ffma2_rn(bc(w4.y), f2(xa.x, xa.y), sc);
          sd = __ffma2_rn(bc(w4.y), f2(xa.z, xa.w), sd);
          sa = __ffma2_rn(bc(w4.z), f2(xb.x, xb.y), sa);
          sb = __ffma2_rn(bc(w4.z), f2(xb.z, xb.w), sb);
          sc = __ffma2_rn(bc(w4.w), f2(xb.x, xb.y), sc);
          sd = __ffma2_rn(bc(w4.w), f2(xb.z, xb.w), sd);
        }
      }
      if constexpr (!COLA) {
        float* sr = Sred + (warp * 8 + 2 * g) * 32 + 4 * q;
        *reinterpret_cast<float4*>(sr) = make_float4(sa.x, sa.y, sb.x, sb.y);
        *reinterpret_cast<float4*>(sr + 32) = make_float4(sc.x, sc.y, sd.x, sd.y);
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NBAR) : "memory");
    // ---- H update: thread handles (k, c) for k in {kt, kt+4}, c = ct
#pragma unroll
    for (int hh = 0; hh < HH; ++hh) {
      const int kt = (tid >> 5) + NW * hh, ct = tid & 31;
      const int64_t col = jt + ct;
      const float hkc = *reinterpret_cast<const float*>(st + XB + kt * 128 + (((ct >> 2) ^ kt) << 4) + (ct & 3) * 4);
      float hn;
      if (do_update) {
        float S = 0.0f;
#pragma unroll
        for (int w = 0; w < NW; ++w) S += Sred[(w * 8 + kt) * 32 + ct];
        float hl[8];
#pragma unroll
        for (int l = 0; l < 8; ++l)
          hl[l] = *reinterpret_cast<const float*>(st + XB + l * 128 + (((ct >> 2) ^ l) << 4) + (ct & 3) * 4);
        if (bcd) {
#pragma unroll
          for (int l = 0; l < 8; ++l) hl[l] *= bsh[l];
        }
        float e0 = 0.0f, e1 = 0.0f;
#pragma unroll
        for (int l = 0; l < 8; l += 2) {
          e0 = fmaf(Gs[kt * 8 + l], hl[l], e0);
          e1 = fmaf(Gs[kt * 8 + l + 1], hl[l + 1], e1);
        }
        if (bcd)  // prox-linear step (Alg. 3 l.14) on H_m = diag(sH) H_m stored
          hn = fmaxf(0.f, fmaf(-((e0 + e1) - S), binvL, hkc * bsh[kt]));
        else
          hn = mu_q(hkc, S, e0 + e1, eps);
        if (kt >= r || col >= n) hn = 0.0f;
        if (kt < r && col < n) Ho[(int64_t)kt * n + col] = hn;
      } else {
        hn = (kt < r && col < n) ? hkc : 0.0f;
      }
      if (do_acc) Hn[hnc_idx(ct, kt)] = hn;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NBAR) : "memory");

    if (do_acc) {
      // ---- phase B
      {
        float qa[QR];
#pragma unroll
        for (int qq = 0; qq < QR; ++qq) qa[qq] = 0.f;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const float* src = Hn + hnc_idx(8 * cs + t, 0);
          const float hr = src[rb];
#pragma unroll
          for (int qq = 0; qq < QR; ++qq) qa[qq] = fmaf(src[QR * warp + qq], hr, qa[qq]);
        }
#pragma unroll
        for (int qq = 0; qq < QR; ++qq) qd[qq] += (double)qa[qq];
      }
#pragma unroll
      for (int h = 0; h < NCH; ++h) {
        float2 acc[16];
#pragma unroll
        for (int v = 0; v < 16; ++v) acc[v] = f2(0.f, 0.f);
#pragma unroll
        for (int s4 = 0; s4 < 2; ++s4) {
          float2 hq2[4][4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float* src = Hn + hnc_idx(8 * cs + 4 * s4 + t, 0);
            const float4 a = *reinterpret_cast<const float4*>(src);
            const float4 bq = *reinterpret_cast<const float4*>(src + 4);
            hq2[t][0] = f2(a.x, a.y);
            hq2[t][1] = f2(a.z, a.w);
            hq2[t][2] = f2(bq.x, bq.y);
            hq2[t][3] = f2(bq.z, bq.w);
          }
          float xs[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = warp * RW + 32 * h + rb + 8 * u;
            const float4 x = lds128(st + i * 128 + (((2 * cs + s4) ^ rb) << 4));
            xs[u][0] = x.x;
            xs[u][1] = x.y;
            xs[u][2] = x.z;
            xs[u][3] = x.w;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int kp = 0; kp < 4; ++kp)
                acc[u * 4 + kp] = __ffma2_rn(bc(xs[u][t]), hq2[t][kp], acc[u * 4 + kp]);
        }
        // reduce-scatter over the 4 column-slice lanes: keep flat f in [8 cs, 8 cs + 8)
        float a1[32];
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          a1[2 * v] = acc[v].x;
          a1[2 * v + 1] = acc[v].y;
        }
        float a2[16];
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const float send = h1 ? a1[v] : a1[v + 16];
          const float keep = h1 ? a1[v + 16] : a1[v];
          a2[v] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const float send = h0 ? a2[v] : a2[v + 8];
          const float keep = h0 ? a2[v + 8] : a2[v];
          accd[h][v] += (double)(keep + __shfl_xor_sync(0xffffffffu, send, 8));
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

  if (do_acc) {
  // P: lane holds flat f = u*8 + k in [8 cs, 8 cs + 8) of sub-chunk h, rows warp*RW + 32h + rb + 8u
  const int mr = m * r, rr = r * r;
  double* Pb = persist ? pa.part + b * (mr + rr) : Ppart + b * mr;
  double* Qb = persist ? pa.part + b * (mr + rr) + mr : Qpart + b * rr;
#pragma unroll
  for (int h = 0; h < NCH; ++h)
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      const int f = 8 * cs + v;
      const int u = f >> 3, k = f & 7;
      const int row = warp * RW + 32 * h + rb + 8 * u;
      if (row < m && k < r) Pb[row * r + k] = accd[h][v];
    }
  // Q rows QR w + qq, column rb: sum the 4 column slices
#pragma unroll
  for (int qq = 0; qq < QR; ++qq) {
    qd[qq] += __shfl_xor_sync(0xffffffffu, qd[qq], 16);
    qd[qq] += __shfl_xor_sync(0xffffffffu, qd[qq], 8);
    if (cs == 0 && rb < r && QR * warp + qq < r) Qb[(QR * warp + qq) * r + rb] = qd[qq];
  }
  }
  }  // consumer warps
  if (!persist || !do_acc) break;
  persist_step(pa, epoch, m, r, eps, Wc, Gs, reinterpret_cast<double*>(stages), it, WPAIR);
  }  // passes
}

size_t fixed_bytes_c(int MP, int NW) {
  return (size_t)NW * 8 * 32 * 4 + 256 + HNC_FLOATS * 4 + (size_t)MP * 8 * 4 + 2 * 16 * 8 + 1024;
}

bool c_one_cta() {  // experiment: NTT_C_1CTA=1 runs the 4-warp variant at 1 CTA / SM with a deeper ring
  static const bool on = [] {
    const char* e = getenv("NTT_C_1CTA");
    return e && e[0] == '1';
  }();
  return on;
}

int stages_c(int MP, int NW) {
  const size_t SB = (size_t)MP * 128 + 1024;
  const size_t budget = (NW == 4 && !c_one_cta()) ? (size_t)SMEM_C : (size_t)SMEM_BUDGET;  // 2 CTAs / SM or 1
  int ns = (int)((budget - fixed_bytes_c(MP, NW)) / SB);
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

template <int MP, int NW>
cudaError_t launch_c(const CUtensorMap& mx, const CUtensorMap& mh, int m, int64_t n, int r, const float* W,
                     const double* Gpart, int nG, float eps, float* H, double* Ppart, double* Qpart, int mode, int grid,
                     int evict_first, const PersistArgs& pa, cudaStream_t st) {
  const int ns = stages_c(MP, NW);
  const size_t SB = (size_t)MP * 128 + 1024;
  const size_t smem = (size_t)ns * SB + fixed_bytes_c(MP, NW);
  cudaError_t e = cudaFuncSetAttribute(k_fused_c<MP, NW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_maybe_coop(k_fused_c<MP, NW>, grid, (NW + 1) * 32, smem, st, pa.iters > 0, mx, mh, m, n, r, W, Gpart,
                           nG, eps, H, Ppart, Qpart, mode, ns, evict_first, pa);
}

// 8 consumer warps, 1 CTA / SM, W rows in registers for m > 128 (NTT_C_NW=4: the 2-CTA variant)
int c_nw(int MP) {
  static const int env = [] {
    const char* e = getenv("NTT_C_NW");
    return e ? atoi(e) : 4;  // the 8-warp variant measured slower (502 vs 362 us/iter, step 2)
  }();
  return (MP == 256 && env == 8) ? 8 : 4;
}

// ===========================================================================
// Variant WC: warp-owned 32-column tiles for 40 < m <= 256 (rank padded to 8),
// no CTA barriers in the loop.  6 consumer warps (<= 2 per SMSP, 255 regs) + 1
// TMA warp; each warp owns `dpw` ring stages (stage = tile's warp * dpw +
// round % dpw), so every warp waits only on rounds it consumed itself.
//   phase A  lanes (q: columns 4q..4q+3, g: ranks 2g, 2g+1) stream all MP rows:
//            X by 128-bit loads, W as row pairs (one 128-bit broadcast per 2 rows)
//   H update lane forms E = G H and Hn for its 2 ranks x 4 columns; 128-bit
//            coalesced stores; Hn into the warp's transposed smem tile
//   phase B  32-row chunks, lanes (rb, cs: 8-column slice), reduce-scatter over
//            the slices, per-lane fp32 accumulators for ALL rows (8 values per
//            chunk) flushed every 32 tiles into the warp's private fp64 global
//            partial (no atomics: deterministic); Q = Hn Hn^T likewise.
// ===========================================================================
constexpr int NWW = 6;
constexpr int NTW = (NWW + 1) * 32;
constexpr int WC_FLUSH = 32;

template <int MP>
__global__ void __launch_bounds__(NTW, 1)
k_fused_wc(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmH, int m, int64_t n, int r,
           const float* __restrict__ W, const double* __restrict__ Gpart, int nG, float eps, float* __restrict__ H,
           double* __restrict__ Ppart, double* __restrict__ Qpart, int mode, int dpw, int evict_first) {
  extern __shared__ unsigned char smem_raw[];
  // keep the shared address space visible to the compiler (LDS/STS, not generic LD/ST)
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  constexpr int NCH = MP / 32;
  constexpr uint32_t XB = MP * 128u;
  constexpr uint32_t SB = XB + 1024u;
  const int ns = NWW * dpw;
  unsigned char* stages = smem;
  float* Wp = reinterpret_cast<float*>(smem + (size_t)ns * SB);  // [MP/2][4 g][4]: W row pairs
  float* Gs = Wp + MP * 8;                                         // 8 x 8
  float* HnAll = Gs + 64;                                          // NWW x HNC_FLOATS
  uint64_t* full = reinterpret_cast<uint64_t*>(HnAll + NWW * HNC_FLOATS);
  uint64_t* empty = full + ns;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool do_update = (mode & kFusedUpdate) != 0;
  const bool do_acc = (mode & kFusedAcc) != 0;
  if (do_update) {
    const int rr = r * r;
    for (int e = tid; e < 64; e += NTW) {
      int k = e >> 3, l = e & 7;
      double sum = 0.0;
      if (k < r && l < r)
        for (int bq = 0; bq < nG; ++bq) sum += Gpart[(int64_t)bq * rr + k * r + l];
      Gs[e] = (float)sum;
    }
  }
  for (int e = tid; e < MP * 8; e += NTW) {
    // Wp[(i/2)*16 + g*4 + (i&1)*2 + t] = W[i][2g + t]
    const int ip = e >> 4, g = (e >> 2) & 3, w2 = e & 3;
    const int i = 2 * ip + (w2 >> 1), k = 2 * g + (w2 & 1);
    Wp[e] = (i < m && k < r) ? W[(int64_t)i * r + k] : 0.0f;
  }
  if (tid == 0) {
    for (int s = 0; s < ns; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int64_t ntiles = (n + BNC - 1) / BNC;
  const int64_t b = blockIdx.x;
  const int64_t J = (ntiles > b) ? (ntiles - b + gridDim.x - 1) / gridDim.x : 0;

  if (warp == NWW) {
    if (lane == 0) {
      uint64_t policy;
      if (evict_first)
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
      else
        asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(policy));
      for (int64_t j = 0; j < J; ++j) {
        const int64_t rnd = j / NWW;
        const int s = (int)(j % NWW) * dpw + (int)(rnd % dpw);
        const uint32_t ph = (uint32_t)((rnd / dpw) & 1);
        MBAR_WAIT(&empty[s], ph ^ 1u, 5, j);
        mbar_expect_tx(&full[s], SB);
        const int col0 = (int)((b + j * gridDim.x) * BNC);
        unsigned char* st = stages + (size_t)s * SB;
        tma_load_2d(st, &tmX, col0, 0, &full[s], policy);
        tma_load_2d(st + XB, &tmH, col0, 0, &full[s], policy);
      }
    }
    return;
  }

  float* Hw = HnAll + warp * HNC_FLOATS;
  const int q = lane & 7, g = lane >> 3;    // phase A / H update
  const int rb = lane & 7, cs = lane >> 3;  // phase B
  const bool h1 = (lane >> 4) & 1, h0 = (lane >> 3) & 1;
  float accf[NCH][8];
  float qf[8];
#pragma unroll
  for (int h = 0; h < NCH; ++h)
#pragma unroll
    for (int v = 0; v < 8; ++v) accf[h][v] = 0.f;
#pragma unroll
  for (int v = 0; v < 8; ++v) qf[v] = 0.f;
  const int mr = m * r, rr = r * r;
  const int64_t slot = b * NWW + warp;  // this warp's private partial
  int nflush = 0, since = 0;
  // flush the fp32 accumulators into the warp's fp64 partial (first flush writes)
  auto flush = [&]() {
#pragma unroll
    for (int h = 0; h < NCH; ++h)
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int f = 8 * cs + v;  // flat u*8 + k within the chunk
        const int u = f >> 3, k = f & 7;
        const int row = 32 * h + rb + 8 * u;
        if (row < m && k < r) {
          double* dst = Ppart + slot * mr + row * r + k;
          *dst = (nflush ? *dst : 0.0) + (double)accf[h][v];
        }
        accf[h][v] = 0.f;
      }
    // Q[rb][l]: sum the 4 column-slice lanes
#pragma unroll
    for (int v = 0; v < 8; ++v) {
      float t = qf[v];
      t += __shfl_xor_sync(0xffffffffu, t, 16);
      t += __shfl_xor_sync(0xffffffffu, t, 8);
      if (cs == 0 && rb < r && v < r) {
        double* dst = Qpart + slot * rr + rb * r + v;
        *dst = (nflush ? *dst : 0.0) + (double)t;
      }
      qf[v] = 0.f;
    }
    ++nflush;
    since = 0;
  };

  for (int64_t j = warp; j < J; j += NWW) {
    const int64_t rnd = j / NWW;
    const int s = warp * dpw + (int)(rnd % dpw);
    const uint32_t ph = (uint32_t)((rnd / dpw) & 1);
    MBAR_WAIT(&full[s], ph, 6, j);
    const unsigned char* st = stages + (size_t)s * SB;
    const int64_t jt = (b + j * gridDim.x) * BNC;
    const int64_t c0 = jt + 4 * q;

    // ---- phase A + H update (lane: ranks 2g, 2g+1 x columns 4q..4q+3)
    // (rows 2g, 2g+1 of the H tile are loaded separately: indexing the hv
    //  register array with the lane-dependent g would spill it to local memory)
    float hk[2][4];
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
      const int k = 2 * g + kk;
      const float4 t4 = lds128(st + XB + k * 128 + ((q ^ k) << 4));
      hk[kk][0] = t4.x; hk[kk][1] = t4.y; hk[kk][2] = t4.z; hk[kk][3] = t4.w;
    }
    float hn[2][4];
    if (do_update) {
      float2 sa = f2(0.f, 0.f), sb = f2(0.f, 0.f), sc = f2(0.f, 0.f), sd = f2(0.f, 0.f);
#pragma unroll 4
      for (int ip = 0; ip < MP / 2; ++ip) {
        const int i = 2 * ip;
        const float4 x0 = lds128(st + i * 128 + ((q ^ (i & 7)) << 4));
        const float4 x1 = lds128(st + (i + 1) * 128 + ((q ^ ((i + 1) & 7)) << 4));
        const float4 wv = *reinterpret_cast<const float4*>(Wp + ip * 16 + g * 4);
        sa = __ffma2_rn(bc(wv.x), f2(x0.x, x0.y), sa);
        sb = __ffma2_rn(bc(wv.x), f2(x0.z, x0.w), sb);
        sc = __ffma2_rn(bc(wv.y), f2(x0.x, x0.y), sc);
        sd = __ffma2_rn(bc(wv.y), f2(x0.z, x0.w), sd);
        sa = __ffma2_rn(bc(wv.z), f2(x1.x, x1.y), sa);
        sb = __ffma2_rn(bc(wv.z), f2(x1.z, x1.w), sb);
        sc = __ffma2_rn(bc(wv.w), f2(x1.x, x1.y), sc);
        sd = __ffma2_rn(bc(wv.w), f2(x1.z, x1.w), sd);
      }
      const float S[2][4] = {{sa.x, sa.y, sb.x, sb.y}, {sc.x, sc.y, sd.x, sd.y}};
      float hv[8][4];
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const float4 t4 = lds128(st + XB + l * 128 + ((q ^ l) << 4));
        hv[l][0] = t4.x; hv[l][1] = t4.y; hv[l][2] = t4.z; hv[l][3] = t4.w;
      }
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const int k = 2 * g + kk;
        float gk[8];
        *reinterpret_cast<float4*>(gk) = *reinterpret_cast<const float4*>(Gs + k * 8);
        *reinterpret_cast<float4*>(gk + 4) = *reinterpret_cast<const float4*>(Gs + k * 8 + 4);
        float2 e01 = f2(0.f, 0.f), e23 = f2(0.f, 0.f);
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          e01 = __ffma2_rn(bc(gk[l]), f2(hv[l][0], hv[l][1]), e01);
          e23 = __ffma2_rn(bc(gk[l]), f2(hv[l][2], hv[l][3]), e23);
        }
        const float e[4] = {e01.x, e01.y, e23.x, e23.y};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float v = mu_q(hk[kk][t], S[kk][t], e[t], eps);
          if (k >= r || c0 + t >= n) v = 0.f;
          hn[kk][t] = v;
        }
        if (k < r) {
          if (c0 + 3 < n) {
            *reinterpret_cast<float4*>(H + (int64_t)k * n + c0) = make_float4(hn[kk][0], hn[kk][1], hn[kk][2], hn[kk][3]);
          } else {
#pragma unroll
            for (int t = 0; t < 4; ++t)
              if (c0 + t < n) H[(int64_t)k * n + c0 + t] = hn[kk][t];
          }
        }
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < 2; ++kk)
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int k = 2 * g + kk;
          hn[kk][t] = (k < r && c0 + t < n) ? hk[kk][t] : 0.f;
        }
    }

    if (do_acc) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        *reinterpret_cast<float2*>(Hw + hnc_idx(4 * q + t, 2 * g)) = f2(hn[0][t], hn[1][t]);
      __syncwarp();
      // ---- Q rows rb over this lane's 8 columns
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const float* src = Hw + hnc_idx(8 * cs + t, 0);
        const float4 a = *reinterpret_cast<const float4*>(src);
        const float4 bq = *reinterpret_cast<const float4*>(src + 4);
        const float hr = src[rb];
        qf[0] = fmaf(hr, a.x, qf[0]); qf[1] = fmaf(hr, a.y, qf[1]);
        qf[2] = fmaf(hr, a.z, qf[2]); qf[3] = fmaf(hr, a.w, qf[3]);
        qf[4] = fmaf(hr, bq.x, qf[4]); qf[5] = fmaf(hr, bq.y, qf[5]);
        qf[6] = fmaf(hr, bq.z, qf[6]); qf[7] = fmaf(hr, bq.w, qf[7]);
      }
      // ---- phase B: P rows in 32-row chunks
#pragma unroll
      for (int h = 0; h < NCH; ++h) {
        float2 acc[16];
#pragma unroll
        for (int v = 0; v < 16; ++v) acc[v] = f2(0.f, 0.f);
#pragma unroll
        for (int s4 = 0; s4 < 2; ++s4) {
          float2 hq2[4][4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float* src = Hw + hnc_idx(8 * cs + 4 * s4 + t, 0);
            const float4 a = *reinterpret_cast<const float4*>(src);
            const float4 bq = *reinterpret_cast<const float4*>(src + 4);
            hq2[t][0] = f2(a.x, a.y);
            hq2[t][1] = f2(a.z, a.w);
            hq2[t][2] = f2(bq.x, bq.y);
            hq2[t][3] = f2(bq.z, bq.w);
          }
          float xs[4][4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int i = 32 * h + rb + 8 * u;
            const float4 x = lds128(st + i * 128 + (((2 * cs + s4) ^ rb) << 4));
            xs[u][0] = x.x; xs[u][1] = x.y; xs[u][2] = x.z; xs[u][3] = x.w;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
              for (int kp = 0; kp < 4; ++kp)
                acc[u * 4 + kp] = __ffma2_rn(bc(xs[u][t]), hq2[t][kp], acc[u * 4 + kp]);
        }
        float a1[32];
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          a1[2 * v] = acc[v].x;
          a1[2 * v + 1] = acc[v].y;
        }
        float a2[16];
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          const float send = h1 ? a1[v] : a1[v + 16];
          const float keep = h1 ? a1[v + 16] : a1[v];
          a2[v] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const float send = h0 ? a2[v] : a2[v + 8];
          const float keep = h0 ? a2[v + 8] : a2[v];
          accf[h][v] += keep + __shfl_xor_sync(0xffffffffu, send, 8);
        }
      }
      if (++since == WC_FLUSH) flush();
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  if (do_acc) flush();  // final (also writes zeros for warps without tiles)
}

size_t fixed_bytes_wc(int MP) {
  return (size_t)MP * 8 * 4 + 256 + (size_t)NWW * HNC_FLOATS * 4 + 2 * 24 * 8 + 1024;
}

int dpw_wc(int MP) {
  const size_t SB = (size_t)MP * 128 + 1024;
  int d = (int)((SMEM_BUDGET - fixed_bytes_wc(MP)) / (SB * NWW));
  return d > 4 ? 4 : d;
}

template <int MP>
cudaError_t launch_wc(const CUtensorMap& mx, const CUtensorMap& mh, int m, int64_t n, int r, const float* W,
                      const double* Gpart, int nG, float eps, float* H, double* Ppart, double* Qpart, int mode, int grid,
                      int evict_first, cudaStream_t st) {
  const int dpw = dpw_wc(MP);
  const size_t SB = (size_t)MP * 128 + 1024;
  const size_t smem = (size_t)NWW * dpw * SB + fixed_bytes_wc(MP);
  cudaError_t e = cudaFuncSetAttribute(k_fused_wc<MP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_fused_wc<MP><<<grid, NTW, smem, st>>>(mx, mh, m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, dpw, evict_first);
  return cudaGetLastError();
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
  cudaError_t e = cudaFuncSetAttribute(k_fused<R, UX, NWT, HD, BNT, FOLD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  return launch_maybe_coop(k_fused<R, UX, NWT, HD, BNT, FOLD>, grid, (NWT + 1) * 32, smem, st, pa.iters > 0, mx, mh,
                           mh2 ? *mh2 : mh, m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, ns, evict_first, pa);
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
  if (m < 1 || m > 256 || r < 1 || r > 8 || n < 4) return false;
  if ((n & 3) || (ldx & 3)) return false;
  if ((reinterpret_cast<uintptr_t>(X) & 15) || (reinterpret_cast<uintptr_t>(H) & 15)) return false;
  if (n > (int64_t)INT32_MAX - 256) return false;
  return true;
}

// Variant WC (warp-owned m <= 256 tiles) is kept as an experiment (NTT_FUSED_WC=1);
// the CTA-cooperative variant C measured faster on config 3 step 2 (DESIGN.md s.6).
bool use_wc() {
  static const bool on = [] {
    const char* e = getenv("NTT_FUSED_WC");
    return e && e[0] == '1';
  }();
  return on;
}

int fused_partials(int64_t m, int64_t n, int r, int num_sms) {
  const int g = fused_grid(m, n, r, num_sms);
  return (m > 40 && use_wc()) ? g * NWW : g;
}

int fused_grid(int64_t m, int64_t n, int r, int num_sms) {
  (void)r;
  if (m <= 40) {
    int64_t ntiles = (n + BN - 1) / BN;
    return (int)(ntiles < num_sms ? ntiles : num_sms);
  }
  int64_t ntiles = (n + BNC - 1) / BNC;
  if (use_wc()) {  // variant WC: one CTA per SM, 6 warp-owned tiles in flight
    int64_t need = (ntiles + NWW - 1) / NWW;
    return (int)(need < num_sms ? (need < 1 ? 1 : need) : num_sms);
  }
  const int cps = (c_nw(m <= 128 ? 128 : 256) == 8 || c_one_cta()) ? 1 : 2;  // variant C: CTAs per SM
  return (int)(ntiles < cps * num_sms ? ntiles : cps * num_sms);
}

size_t fused_scratch_bytes(int64_t, int64_t, int, int) { return 0; }
void fused_destroy(FusedCtx&) {}

struct FusedPlan {
  bool x3d;  // X (and staged H) through 3-D maps: one box per 128-column tile
  bool hd;   // lanes load H directly (no H boxes in the stage)
  int bn;    // tile width (columns)
};

// the k_fused variant launch_fused picks for m <= 40 (environment knobs: DESIGN.md s.6)
FusedPlan fused_plan(int64_t m, int64_t n, int r) {
  static const bool x3d_on = [] {
    const char* e = getenv("NTT_X3D");
    const char* b = getenv("NTT_W_BN");  // the 3-D box spans 4 blocks: 128-column tiles only
    return !(e && e[0] == '0') && !(b && b[0] == '6');
  }();
  static const int x3d_max_ux = [] {
    const char* e = getenv("NTT_X3D_UX");
    return e ? atoi(e) : 5;
  }();
  // experiment knobs: NTT_W_BN=64 (64-column tiles for UX >= 4), NTT_W_HDIRECT=0/1 (default: direct H loads
  // when m <= 16 or r < 8, i.e. when H is a large share of the traffic)
  static const int w_bn = [] {
    const char* e = getenv("NTT_W_BN");
    return (e && e[0] == '6') ? 64 : 128;
  }();
  static const int w_hd = [] {
    const char* e = getenv("NTT_W_HDIRECT");
    return e ? (e[0] == '1' ? 1 : 0) : -1;
  }();
  const int ux = ux_for(m);
  FusedPlan p;
  p.x3d = ux <= x3d_max_ux && (n % 32) == 0 && x3d_on;
  // with the 3-D maps staging H through TMA (one 4 KB box per tile) beats the lanes' direct
  // loads, which cannot keep enough bytes in flight (tools/membench.cu): config 4 step 1
  // 59.4 -> 53.7 ms, steps 2-5 -2 to -5 %
  p.hd = (w_hd >= 0) ? (w_hd == 1) : (p.x3d ? false : (ux <= 2 || r < 8));
  p.bn = (ux >= 4 && w_bn == 64) ? 64 : 128;
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
  if (pa.iters > 0 && m > 40 && use_wc()) return cudaErrorNotSupported;
  const int evict_first = ((double)m * (double)n * 4.0 > 48e6) ? 1 : 0;
  if (m > 40 && use_wc()) {
    const int MPc = m <= 128 ? 128 : 256;
    CUtensorMap mx, mh;
    cudaError_t e = make_map(&mx, X, (uint64_t)n, (uint64_t)m, (uint64_t)ldx, (uint32_t)MPc);
    if (e != cudaSuccess) return e;
    e = make_map(&mh, H, (uint64_t)n, (uint64_t)r, (uint64_t)n, 8u);
    if (e != cudaSuccess) return e;
    if (MPc == 128) return launch_wc<128>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, evict_first, st);
    return launch_wc<256>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, evict_first, st);
  }
  if (m > 40) {
    const int MPc = m <= 128 ? 128 : 256;
    CUtensorMap mx, mh;
    cudaError_t e = make_map(&mx, X, (uint64_t)n, (uint64_t)m, (uint64_t)ldx, (uint32_t)MPc);
    if (e != cudaSuccess) return e;
    e = make_map(&mh, H, (uint64_t)n, (uint64_t)r, (uint64_t)n, 8u);
    if (e != cudaSuccess) return e;
    if (MPc == 128) return launch_c<128, 4>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, evict_first, pa, st);
    if (c_nw(256) == 8)
      return launch_c<256, 8>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, evict_first, pa, st);
    return launch_c<256, 4>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, evict_first, pa, st);
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
  const int w_bn = fp.bn;
  const bool hd = fp.hd;
  // H boxes (staged path): 3-D as well when X uses the 3-D map (block stride 128 B of row pitch n)
  auto hmap = [&](CUtensorMap* mp, const float* base) {
    return (ef & 2) && !hd && (n % 32) == 0 ? make_map3(mp, base, (uint64_t)n, (uint64_t)r, (uint64_t)n, 8u, 4u)
                                            : make_map(mp, base, (uint64_t)n, (uint64_t)r, (uint64_t)n, 8u);
  };
  e = hmap(&mh, H);
  if (e != cudaSuccess) return e;
  if (pa.bcdFold) {  // BCD H_m fold: both H buffers (fused_fold_ok() said this variant runs)
    if (hd || w_bn != 128 || !pa.Hout || !pa.Hout2 || !pa.bcdRole) return cudaErrorNotSupported;
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
#define LF(RR, UU)                                                                                                              \
  return (UU >= 4 && w_bn == 64)                                                                                                  \
             ? (hd ? launch_t<RR, UU, 8, true, 64>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, ef, pa, st)  \
                   : launch_t<RR, UU, 8, false, 64>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, ef, pa, st)) \
             : (hd ? launch_t<RR, UU, 8, true, 128>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, ef, pa, st) \
                   : launch_t<RR, UU, 8, false, 128>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, ef, pa, st))
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
  static const int w_nwt = [] {
    const char* e = getenv("NTT_W_NWT");
    return e ? atoi(e) : 8;
  }();
  if (ux == 4 && !hd && w_bn == 128 && w_nwt == 6)
    return launch_t<8, 4, 6, false, 128>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, ef, pa, st);
  if (ux == 4 && !hd && w_bn == 128 && w_nwt == 9)
    return launch_t<8, 4, 9, false, 128>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, ef, pa, st);
  if (ux == 4 && !hd && w_bn == 128 && w_nwt == 7)
    return launch_t<8, 4, 7, false, 128>(mx, mh, (int)m, n, r, W, Gpart, nG, eps, H, Ppart, Qpart, mode, grid, ef, pa, st);
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
