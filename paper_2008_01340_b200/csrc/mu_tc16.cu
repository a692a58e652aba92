// mu_tc16.cu -- fp16x2 variant of the tensor-core 2-pass MU iteration (mu_tc.cu).
//
// A tcgen05 MMA with M = 128 costs ~138 cycles per instruction for any N <= 128
// (tools/tc_probe.cu), and an instruction consumes 32 bytes of K per A row: 8 tf32
// or 16 fp16 elements.  Splitting operands into two fp16 parts instead of two tf32
// parts therefore halves the MMA count per X element:
//   v * s = v0 + v1,  v0 = fp16(v s),  v1 = fp16(v s - v0)      (~22 significant bits)
//   D[:, 0:2R] (+)= A0 * [B0 | B1],   D[:, 0:R] += A1 * B0        (kind::f16, fp32 accumulate)
// with per-tensor power-of-two scales s (X: once per call from max|X|; W, H: at
// every update from their max) chosen so that max |v s| < 2^14 (no fp16 overflow);
// the epilogue multiplies by 1 / (s_X s_F) exactly.  For non-negative data (every
// MU operand) there is no cancellation, so the parts' ~2^-22 relative error and the
// 2^-24 absolute floor of fp16 subnormals stay far below the 1e-4 parity bar.
// Both A parts are staged in TMEM by the converter warps; B = [B0; B1] (fp16, 2R x K,
// K-major, SWIZZLE_128B) is written by the pack kernels.  Pipeline, split-K
// partials and fp64 flushes are those of k_skinny_tc (mu_tc.cu).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "mu_tc.h"
#include "sm100.cuh"

namespace ntt {

namespace {
using namespace sm100;

constexpr int T16_BK = 64;      // K elements per stage (fp32 X: two 128-B rows; fp16 B: one 128-B row)
constexpr int T16_BM = 128;
constexpr int T16_T = 4;        // TMEM A buffers (each: A0 32 cols + A1 32 cols)
constexpr int T16_THREADS = 320;
constexpr uint32_t T16_ABYTES = T16_BM * T16_BK * 4u;  // 32 KB

template <int R>
struct T16Cfg {
  static constexpr int N1 = 2 * R;
  static constexpr uint32_t BBYTES = (uint32_t)N1 * 128u;  // 64 fp16 per row
  static constexpr uint32_t SB = T16_ABYTES + BBYTES;
  static constexpr uint32_t TMEM_D = 0;
  static constexpr uint32_t TMEM_A = 2 * N1;  // T16_T buffers x 64 columns
  static constexpr uint32_t TMEM_COLS = 512u;
};

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4)                       // c_format = F32; a/b format 0 = F16
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// split (a, b) = (K index 2p, 2p + 1) into packed hi / lo fp16 pairs (low half = lower K)
// (packed fp32x2 / f16x2 conversions: per component the same IEEE round-to-nearest operations as
// the scalar form -- scale, round to fp16, exact back-conversion, subtract, round -- so the parts
// are bit-identical; half the converter-warp instructions)
__device__ __forceinline__ void split2(float a, float b, float s, uint32_t& hi, uint32_t& lo) {
  const float2 v = __fmul2_rn(make_float2(a, b), make_float2(s, s));
  const __half2 h = __floats2half2_rn(v.x, v.y);
  const float2 hf = __half22float2(h);
  const float2 d = __fadd2_rn(v, make_float2(-hf.x, -hf.y));
  const __half2 l = __floats2half2_rn(d.x, d.y);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}

// MODE 0: D (Mtot = m) = X Bcat^T, A = X rows: two [128 rows][32 cols] boxes per stage.
// MODE 1: D (Mtot = n) = X^T Bcat^T, A = X^T: four [64 K rows][32 cols] boxes per stage.
// scales[0] = s_X, scales[1 + MODE ? ...]: sF at scales[sidx]; epilogue multiplies by 1/(s_X sF).
template <int R, int MODE>
__global__ void __launch_bounds__(T16_THREADS, 1)
k_skinny_tc16(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int64_t Mtot,
              int64_t ktiles, int nsplit, int64_t kchunk, int ns, int flush, int r, double* __restrict__ part,
              const float* __restrict__ scales, int sidx, int evict_first) {
  using C = T16Cfg<R>;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)ns * C::SB);
  uint64_t* empty = full + ns;
  uint64_t* a_full = empty + ns;
  uint64_t* a_empty = a_full + T16_T;
  uint64_t* acc_full = a_empty + T16_T;
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
    for (int t = 0; t < T16_T; ++t) {
      mbar_init(&a_full[t], 4);
      mbar_init(&a_empty[t], 1);
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
  const int64_t nmb = (Mtot + T16_BM - 1) / T16_BM;
  const int64_t nunits = nmb * nsplit;

  if (warp == 0) {
    // ======================= TMA producer =======================
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      const uint64_t pol = evict_first ? policy_evict_first() : policy_evict_normal();
      const uint64_t polB = policy_evict_normal();
      int s = 0;
      uint32_t ph = 0;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int64_t mb = u / nsplit, sp = u % nsplit;
        const int64_t k0 = sp * kchunk, k1 = ((k0 + kchunk < ktiles) ? k0 + kchunk : ktiles);
        for (int64_t kt = k0; kt < k1; ++kt, s = (s + 1 == ns) ? 0 : s + 1, ph ^= (s == 0) ? 1u : 0u) {
          mbar_wait(&empty[s], ph ^ 1u);
          mbar_expect_tx(&full[s], C::SB);
          unsigned char* st = smem + (size_t)s * C::SB;
          if (MODE == 0) {
            tma_load_2d(st, &tmA, (int)(kt * T16_BK), (int)(mb * T16_BM), &full[s], pol);
            tma_load_2d(st + 16384, &tmA, (int)(kt * T16_BK + 32), (int)(mb * T16_BM), &full[s], pol);
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              tma_load_2d(st + q * 8192, &tmA, (int)(mb * T16_BM + 32 * q), (int)(kt * T16_BK), &full[s], pol);
          }
          tma_load_2d(st + T16_ABYTES, &tmB, (int)(kt * T16_BK), 0, &full[s], polB);
        }
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer =======================
    if (lane == 0) {
      constexpr uint32_t id1 = idesc_f16(T16_BM, C::N1);
      constexpr uint32_t id2 = idesc_f16(T16_BM, R);
      int64_t g = 0;
      int s = 0, t = 0;
      uint32_t ph = 0, pht = 0;
      for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
        const int64_t sp = u % nsplit;
        const int64_t k0 = sp * kchunk, k1 = ((k0 + kchunk < ktiles) ? k0 + kchunk : ktiles);
        for (int64_t kt = k0; kt < k1; ++kt, s = (s + 1 == ns) ? 0 : s + 1, ph ^= (s == 0) ? 1u : 0u,
                     t = (t + 1) & (T16_T - 1), pht ^= (t == 0) ? 1u : 0u) {
          const int64_t i = kt - k0;
          const bool gfirst = (i % flush) == 0;
          const bool glast = ((i + 1) % flush) == 0 || kt + 1 == k1;
          const int a = (int)(g & 1);
          if (gfirst) {
            mbar_wait(&acc_empty[a], (uint32_t)(((g >> 1) & 1) ^ 1));
            tc_fence_after();
          }
          mbar_wait(&full[s], ph);
          mbar_wait(&a_full[t], pht);
          tc_fence_after();
          const uint32_t sb = smem_u32(smem + (size_t)s * C::SB) + T16_ABYTES;
          const uint32_t dcol = tbase + C::TMEM_D + (uint32_t)a * C::N1;
          const uint32_t at = tbase + C::TMEM_A + (uint32_t)t * 64;
#pragma unroll
          for (int kk = 0; kk < T16_BK / 16; ++kk) {
            const uint64_t bdesc = umma_desc_sw128(sb + kk * 32, 16, 1024);
            mma_f16_ts(dcol, at + kk * 8, bdesc, id1, (gfirst && kk == 0) ? 0u : 1u);   // A0 * [B0 | B1]
            mma_f16_ts(dcol, at + 32 + kk * 8, bdesc, id2, 1u);                       // A1 * B0
          }
          mma_commit(&empty[s]);
          mma_commit(&a_empty[t]);
          if (glast) {
            mma_commit(&acc_full[a]);
            ++g;
          }
        }
      }
    }
  } else if (warp < 6) {
    // ======================= converters: A0 / A1 (fp16 pairs) -> TMEM =======================
    const int q = warp & 3;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    const float sx = scales[0];
    int s = 0, t = 0;
    uint32_t ph = 0, pht = 0;
    for (int64_t u = blockIdx.x; u < nunits; u += gridDim.x) {
      const int64_t sp = u % nsplit;
      const int64_t k0 = sp * kchunk, k1 = ((k0 + kchunk < ktiles) ? k0 + kchunk : ktiles);
      for (int64_t kt = k0; kt < k1; ++kt, s = (s + 1 == ns) ? 0 : s + 1, ph ^= (s == 0) ? 1u : 0u,
                   t = (t + 1) & (T16_T - 1), pht ^= (t == 0) ? 1u : 0u) {
        mbar_wait(&full[s], ph);
        mbar_wait(&a_empty[t], pht ^ 1u);
        tc_fence_after();
        const unsigned char* st = smem + (size_t)s * C::SB;
        uint32_t hi[32], lo[32];
        if (MODE == 0) {
          const int rho = 32 * q + lane;
#pragma unroll
          for (int hbox = 0; hbox < 2; ++hbox) {
            const unsigned char* row = st + hbox * 16384 + rho * 128;
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const float4 x = *reinterpret_cast<const float4*>(row + ((ch ^ (rho & 7)) << 4));
              const int p0 = 16 * hbox + 2 * ch;  // pair index of K = 32 hbox + 4 ch
              split2(x.x, x.y, sx, hi[p0], lo[p0]);
              split2(x.z, x.w, sx, hi[p0 + 1], lo[p0 + 1]);
            }
          }
        } else {
          const unsigned char* box = st + q * 8192 + (lane & 3) * 4;
          const int chk = lane >> 2;
#pragma unroll
          for (int i = 0; i < 64; i += 2) {
            const float a = *reinterpret_cast<const float*>(box + i * 128 + ((chk ^ (i & 7)) << 4));
            const float b = *reinterpret_cast<const float*>(box + (i + 1) * 128 + ((chk ^ ((i + 1) & 7)) << 4));
            split2(a, b, sx, hi[i >> 1], lo[i >> 1]);
          }
        }
        tmem_st32(tbase + C::TMEM_A + (uint32_t)t * 64 + lane_off, hi);
        tmem_st32(tbase + C::TMEM_A + (uint32_t)t * 64 + 32 + lane_off, lo);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&a_full[t]);
      }
    }
  } else {
    // ======================= epilogue =======================
    const int q = warp & 3;
    const uint32_t lane_off = (uint32_t)(32 * q) << 16;
    const double inv = 1.0 / ((double)scales[0] * (double)scales[sidx]);
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
          uint32_t vh[16], vl[16];
          tmem_ld16(d + c0, vh);
          tmem_ld16(d + R + c0, vl);
          tmem_ld_wait();
#pragma unroll
          for (int k = 0; k < 16; ++k) acc[c0 + k] += (double)__uint_as_float(vh[k]) + (double)__uint_as_float(vl[k]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[a]);
      }
      const int64_t row = mb * T16_BM + 32 * q + lane;
      if (row < Mtot) {
        double* dst = part + ((int64_t)sp * Mtot + row) * r;
#pragma unroll
        for (int k = 0; k < R; ++k)
          if (k < r) dst[k] = acc[k] * inv;
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

// max |v| over a strided matrix (rows x cols, row stride ld) as float bits (atomicMax on
// non-negative floats orders like their bit patterns; order-independent => deterministic)
__global__ void k_absmax(const float* __restrict__ v, int64_t rows, int64_t cols, int64_t ld,
                         unsigned* __restrict__ out) {
  float mx = 0.0f;
  if (ld == cols) {  // contiguous: one flat grid-stride loop
    const int64_t total = rows * cols;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x)
      mx = fmaxf(mx, fabsf(v[e]));
  } else if (cols >= 128) {  // rows strided over CTAs, columns over threads (coalesced, no division per element)
    for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
      const float* row = v + i * ld;
      for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mx = fmaxf(mx, fabsf(row[j]));
    }
  } else {
    const int64_t total = rows * cols;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = e / cols, j = e - i * cols;
      mx = fmaxf(mx, fabsf(v[i * ld + j]));
    }
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(mx));
}

__device__ __forceinline__ float pow2_scale(unsigned maxbits) {
  const float mx = __uint_as_float(maxbits);
  if (!(mx > 0.0f)) return 1.0f;
  int e;
  frexpf(mx, &e);                 // mx < 2^e
  return ldexpf(1.0f, 14 - e);    // mx * s < 2^14
}

// fp16 parts of a factor: F is r x n (H, row-major, ld n) or m x r (W, then transposed):
// dst[k][j] = fp16(F[k][j] s), dst[R + k][j] = fp16(F[k][j] s - hi); scales[sidx] = s
__global__ void k_pack16(const float* __restrict__ F, int r, int64_t len, bool transposed, int R,
                         const unsigned* __restrict__ maxbits, __half* __restrict__ dst, int64_t ldd,
                         float* __restrict__ scales, int sidx, unsigned* __restrict__ reset) {
  const float s = pow2_scale(*maxbits);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    scales[sidx] = s;
    *reset = 0u;  // the next update's max slot (the other parity)
  }
  // j (the long index) over threads / CTAs, k in an inner loop over this CTA row's chunk of 8
  // ranks (blockIdx.y): no division per element, and r / 8 times the threads of one k loop
  const int k0 = 8 * blockIdx.y, k1 = min(r, k0 + 8);
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < len; j += (int64_t)gridDim.x * blockDim.x) {
    for (int k = k0; k < k1; ++k) {
      const float v = (transposed ? F[j * r + k] : F[(int64_t)k * len + j]) * s;
      const __half h = __float2half_rn(v);
      dst[(int64_t)k * ldd + j] = h;
      dst[(int64_t)(R + k) * ldd + j] = __float2half_rn(v - __half2float(h));
    }
  }
}

__global__ void k_scale_init(float* scales, const unsigned* maxbits) {
  if (threadIdx.x == 0) scales[0] = pow2_scale(*maxbits);
}

PFN_cuTensorMapEncodeTiled_v12000 g_enc16 = nullptr;

cudaError_t enc16() {
  if (g_enc16) return cudaSuccess;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr);
  if (e != cudaSuccess) return e;
  if (qr != cudaDriverEntryPointSuccess || !fn) return cudaErrorNotSupported;
  g_enc16 = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return cudaSuccess;
}

cudaError_t map2d_t(CUtensorMap* map, CUtensorMapDataType dt, size_t esz, const void* base, uint64_t cols,
                    uint64_t rows, uint64_t ld, uint32_t bc, uint32_t br) {
  cudaError_t e = enc16();
  if (e != cudaSuccess) return e;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld * esz};
  cuuint32_t box[2] = {bc, br};
  cuuint32_t es[2] = {1, 1};
  CUresult res = g_enc16(map, dt, 2, const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return res == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int R>
int t16_stages() {
  int s = (int)((227u * 1024u - 2048u) / T16Cfg<R>::SB);
  return std::min(s, 8);
}

template <int R, int MODE>
cudaError_t launch16(const CUtensorMap& ma, const CUtensorMap& mb, int64_t Mtot, int64_t ktiles, int nsplit,
                     int64_t kchunk, int grid, int r, double* part, const float* scales, int sidx, int ef,
                     cudaStream_t st, int flush) {
  const int ns = t16_stages<R>();
  const size_t sm = (size_t)ns * T16Cfg<R>::SB + 2048;
  cudaError_t e = smem_optin((const void*)(k_skinny_tc16<R, MODE>), sm);
  if (e != cudaSuccess) return e;
  k_skinny_tc16<R, MODE><<<grid, T16_THREADS, sm, st>>>(ma, mb, Mtot, ktiles, nsplit, kchunk, ns, flush, r, part,
                                                        scales, sidx, ef);
  return cudaGetLastError();
}

}  // namespace

// ------------------------------------------------------------------ host API
cudaError_t tc16_prepare(const TcPlan& p, const float* X, int64_t ldx, float* H, char* ws, TcMaps* maps,
                         cudaStream_t st) {
  __half* H16 = reinterpret_cast<__half*>(ws + p.off_h16);
  __half* W16 = reinterpret_cast<__half*>(ws + p.off_w16);
  float* scales = reinterpret_cast<float*>(ws + p.off_scales);
  unsigned* mx = reinterpret_cast<unsigned*>(ws + p.off_scales + 64);
  const uint32_t N1 = 2u * (uint32_t)p.R;
  cudaError_t e;
  if ((e = map2d_t(&maps->xw16, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, X, p.n, p.m, ldx, 32, T16_BM))) return e;
  if ((e = map2d_t(&maps->xh16, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, X, p.n, p.m, ldx, 32, 64))) return e;
  if ((e = map2d_t(&maps->hcat16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, H16, p.n, N1, p.ldh16, 64, N1))) return e;
  if ((e = map2d_t(&maps->wcat16, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, W16, p.m, N1, p.ldw16, 64, N1))) return e;
  if ((e = cudaMemsetAsync(H16, 0, sizeof(__half) * (size_t)N1 * p.ldh16, st))) return e;
  if ((e = cudaMemsetAsync(W16, 0, sizeof(__half) * (size_t)N1 * p.ldw16, st))) return e;
  if ((e = cudaMemsetAsync(mx, 0, 32, st))) return e;
  k_absmax<<<4 * p.grid, 256, 0, st>>>(X, p.m, p.n, ldx, mx);
  k_scale_init<<<1, 32, 0, st>>>(scales, mx);
  return cudaGetLastError();
}

// fp16 parts of H (r x n) -> Hcat16, scale at scales[1].  it = -1: the initial H (its max
// is computed here); otherwise k_tc_hupdate of iteration `it` left max|H| in slot 1 + (it & 1).
cudaError_t tc16_pack_h(const TcPlan& p, const float* H, char* ws, cudaStream_t st, int it) {
  unsigned* mx = reinterpret_cast<unsigned*>(ws + p.off_scales + 64);
  unsigned* cur = mx + 1 + (it & 1);
  if (it < 0) {
    k_absmax<<<2 * p.grid, 256, 0, st>>>(H, p.r, p.n, p.n, cur);
    cudaError_t e = cudaGetLastError();
    if (e) return e;
  }
  k_pack16<<<dim3(4 * p.grid, (p.r + 7) / 8), 256, 0, st>>>(H, p.r, p.n, false, p.R, cur, reinterpret_cast<__half*>(ws + p.off_h16), p.ldh16,
                                       reinterpret_cast<float*>(ws + p.off_scales), 1, mx + 1 + ((it + 1) & 1));
  return cudaGetLastError();
}

// fp16 parts of W (m x r) transposed -> WcatT16, scale at scales[2]; max|W| from k_tc_wupdate
cudaError_t tc16_pack_w(const TcPlan& p, const float* W, char* ws, cudaStream_t st, int it) {
  unsigned* mx = reinterpret_cast<unsigned*>(ws + p.off_scales + 64);
  k_pack16<<<dim3(4 * p.grid, (p.r + 7) / 8), 256, 0, st>>>(W, p.r, p.m, true, p.R, mx + 3 + (it & 1),
                                       reinterpret_cast<__half*>(ws + p.off_w16), p.ldw16,
                                       reinterpret_cast<float*>(ws + p.off_scales), 2, mx + 3 + ((it + 1) & 1));
  return cudaGetLastError();
}

// BCD (bcd.cu) slots: 5 = max H (k_bcd_hup), 6 = max W (k_bcd_wnorm), both cleared by
// k_bcd_decide; 7 = the self-contained "fresh" packs below; 4 = a reset target nobody reads
// while BCD runs (the MU W slot, unused there).
unsigned* tc16_max_slot(const TcPlan& p, char* ws, int slot) {
  return reinterpret_cast<unsigned*>(ws + p.off_scales + 64) + slot;
}

cudaError_t tc16_pack_h_slot(const TcPlan& p, const float* H, char* ws, cudaStream_t st, int slot) {
  k_pack16<<<dim3(4 * p.grid, (p.r + 7) / 8), 256, 0, st>>>(H, p.r, p.n, false, p.R, tc16_max_slot(p, ws, slot),
                                       reinterpret_cast<__half*>(ws + p.off_h16), p.ldh16,
                                       reinterpret_cast<float*>(ws + p.off_scales), 1, tc16_max_slot(p, ws, 4));
  return cudaGetLastError();
}

cudaError_t tc16_pack_w_slot(const TcPlan& p, const float* W, char* ws, cudaStream_t st, int slot) {
  k_pack16<<<dim3(4 * p.grid, (p.r + 7) / 8), 256, 0, st>>>(W, p.r, p.m, true, p.R, tc16_max_slot(p, ws, slot),
                                       reinterpret_cast<__half*>(ws + p.off_w16), p.ldw16,
                                       reinterpret_cast<float*>(ws + p.off_scales), 2, tc16_max_slot(p, ws, 4));
  return cudaGetLastError();
}

// fp16 parts of an arbitrary factor with its max computed here (slot 7, cleared first)
cudaError_t tc16_pack_h_fresh(const TcPlan& p, const float* H, char* ws, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(tc16_max_slot(p, ws, 7), 0, sizeof(unsigned), st);
  if (e) return e;
  k_absmax<<<2 * p.grid, 256, 0, st>>>(H, 1, (int64_t)p.r * p.n, (int64_t)p.r * p.n, tc16_max_slot(p, ws, 7));
  return tc16_pack_h_slot(p, H, ws, st, 7);
}

cudaError_t tc16_pass_w(const TcPlan& p, const TcMaps& mp, char* ws, int ef, cudaStream_t st, int flush) {
  double* P = reinterpret_cast<double*>(ws + p.off_P);
  const float* sc = reinterpret_cast<const float*>(ws + p.off_scales);
  const int64_t kt = (p.n + T16_BK - 1) / T16_BK;
  if (p.R == 16) return launch16<16, 0>(mp.xw16, mp.hcat16, p.m, kt, p.splitW16, p.kchW16, p.grid, p.r, P, sc, 1, ef, st, flush);
  return launch16<32, 0>(mp.xw16, mp.hcat16, p.m, kt, p.splitW16, p.kchW16, p.grid, p.r, P, sc, 1, ef, st, flush);
}

cudaError_t tc16_pass_h(const TcPlan& p, const TcMaps& mp, char* ws, int ef, cudaStream_t st, int flush) {
  double* S = reinterpret_cast<double*>(ws + p.off_S);
  const float* sc = reinterpret_cast<const float*>(ws + p.off_scales);
  const int64_t kt = (p.m + T16_BK - 1) / T16_BK;
  if (p.R == 16) return launch16<16, 1>(mp.xh16, mp.wcat16, p.n, kt, p.splitH16, p.kchH16, p.grid, p.r, S, sc, 2, ef, st, flush);
  return launch16<32, 1>(mp.xh16, mp.wcat16, p.n, kt, p.splitH16, p.kchH16, p.grid, p.r, S, sc, 2, ef, st, flush);
}

}  // namespace ntt
