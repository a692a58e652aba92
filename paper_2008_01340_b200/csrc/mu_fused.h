// mu_fused.h -- the 1-pass fused short-wide MU kernel (mu_fused.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ntt {

struct FusedCtx {
  int dummy = 0;
};

// Shapes the TMA-fed warp-tile kernel handles: m <= 40 rows, r <= 8, rows of
// X and H 16-byte aligned (ldx % 4 == 0, n % 4 == 0).
bool fused_supported(int64_t m, int64_t n, int r, int64_t ldx, const void* X, const void* H);
int fused_grid(int64_t m, int64_t n, int r, int num_sms);
// number of (P, Q) partial slots one fused pass writes (>= grid)
int fused_partials(int64_t m, int64_t n, int r, int num_sms);
size_t fused_scratch_bytes(int64_t m, int64_t n, int r, int grid);
void fused_destroy(FusedCtx& c);

// mode bits of one fused pass over X
constexpr int kFusedUpdate = 1;  // phase A: S = W^T X, H <- H o S / (G H + eps), store H
constexpr int kFusedAcc = 2;     // phase B: per-CTA partials of P = X Hn^T, Q = Hn Hn^T

// Persistent mode (iters > 0): one cooperative launch runs the acc-only prologue
// and `iters` fused passes of a TT step, reducing the per-CTA partials and
// updating W inside the kernel (mu_fused.cu, persist_step).  part: [grid][m r + r r]
// fp64, red: [m r + r r] fp64, ctr: zeroed grid-barrier counter, Wout: W (m x r).
struct PersistArgs {
  int iters;
  double* part;
  double* red;
  unsigned* ctr;
  float* Wout;
  unsigned long long* trace;  // nullable: per pass 4 globaltimer stamps of CTA 0 (diagnostics)
  // BCD H step instead of the MU rule (non-persistent k_fused, m <= 40; bcd.cu, Alg. 3 l.11-14):
  // H is then H_m (rows scaled by bcdS[k]) and Hn = max(0, H_m - (G H_m - W^T X) / *bcdL) is
  // stored to Hout (P, Q partials of Hn as usual)
  const double* bcdL = nullptr;
  const double* bcdS = nullptr;
  float* Hout = nullptr;
  float* Hout2 = nullptr;           // with bcdRole: Hn goes to (*bcdRole != 0 ? Hout2 : Hout)
  const double* bcdRole = nullptr;
  // with bcdRole: H_m = diag(bcdS[0..r)) B[1 - role] - diag(bcdS[64..64+r)) B[role], B = (Hout,
  // Hout2), formed inside the pass (k_fused with staged H only; see fused_fold_ok)
  bool bcdFold = false;
  // persistent k_fused_c (40 < m <= 256): X as fp16 hi / lo parts, written by the prologue pass and
  // streamed by every later pass instead of converting the fp32 tile again (fused_x16_bytes;
  // nullable: every pass converts)
  unsigned char* x16 = nullptr;
  // dynamic tail (persistent k_fused_m; the per-SM pass-time spread is systematic, DESIGN s.6): the
  // last tail_groups groups of 16 tiles of every pass are claimed at run time through a counter in
  // ctr[8..9] (one failing claim per CTA per pass); the warp that serves members u, u + 8, ... of group
  // g adds them into partial slot gridDim.x + 8 g + u of part (fixed grouping -> deterministic sums)
  // and parks its static accumulators in park[cta][warp][320] meanwhile.  0 = static schedule.
  int tail_groups = 0;
  double* park = nullptr;
  // cross-GPU exchange (persistent launch on an ntt_create_dist handle, SURVEY s.8(e)): after the
  // per-GPU reduction of every pass, CTA 0 stores the (P, Q) vector into slot [seq & 1][rank] of
  // every rank's exchange buffer (NVLink peer stores; IPC-mapped, own buffer included), raises
  // flag [seq & 1][rank] there with a release store, waits for the nranks flags of its own
  // buffer, and every CTA then sums the nranks slots in rank order (the same sum on every rank).
  // seq: a per-buffer pass counter kept on the device (read at launch, advanced by `iters`).
  // nranks = 0: single-GPU reduction only.
  double* const* xpeers = nullptr;  // [nranks] exchange buffer bases (device array)
  int nranks = 0;
  int rank = 0;
};
// exchange buffer layout (doubles): slots [2][nranks][kXLmax], flags (u64) [2][nranks], seq (u64)
constexpr int kXLmax = 256 * 16 + 16 * 16;  // largest m r + r r of the persistent kernels
__host__ __device__ inline size_t xbuf_bytes(int nranks) {
  return sizeof(double) * 2 * (size_t)nranks * kXLmax + sizeof(unsigned long long) * (2 * (size_t)nranks + 8);
}
// bytes of the PersistArgs::x16 cache for an m x n X (0 when m <= 40)
size_t fused_x16_bytes(int64_t m, int64_t n);
// groups of 16 tiles served dynamically at the end of every pass of the persistent k_fused_m
// (0 = static schedule); the launcher needs pa.part with grid + 8 groups slots and pa.park with
// grid * 8 * 320 doubles
int fused_tail_groups(int64_t m, int64_t n, int r, int grid);

// One pass over X (m x n, row stride ldx) with the current W (m x r) and
// G = sum_c Gpart[c] (nG partials).  mode = kFusedAcc alone is the prologue
// (Hn := H).  Ppart/Qpart: [grid][m*r] / [grid][r*r] fp64.
// whether launch_fused runs the BCD H_m fold (PersistArgs::bcdFold) for this shape and buffers
bool fused_fold_ok(int64_t m, int64_t n, int r, int64_t ldx, const void* X, const void* H0, const void* H1);

cudaError_t launch_fused(const float* X, int64_t ldx, int64_t m, int64_t n, int r, const float* W,
                         const double* Gpart, int nG, float eps, float* H, double* Ppart, double* Qpart, int mode,
                         int grid, cudaStream_t st, const PersistArgs* persist = nullptr);

// W update from partials with a parallel fixed-order reduction:
//   P = sum_b Ppart[b] (nP), Q = sum_b Qpart[b] (nQ), W <- W o P / (W Q + eps);
//   Gpart[c] = sum over CTA c's rows of Wn^T Wn.  Returns the CTA count via *nG.
int wupdate2_ctas(int64_t m, int r);
cudaError_t launch_wupdate2(float* W, int64_t m, int r, const double* Ppart, int nP, const double* Qpart, int nQ,
                            float eps, double* Gpart, cudaStream_t st);

}  // namespace ntt
