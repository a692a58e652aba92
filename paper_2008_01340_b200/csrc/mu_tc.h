// mu_tc.h -- tensor-core (tcgen05 kind::tf32, 3xTF32) 2-pass MU iteration for
// tall / square X (mu_tc.cu).  Internal to libntt.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ntt {

struct TcPlan {
  int64_t m = 0, n = 0;
  int r = 0, R = 0;      // rank and its padded class (16 or 32)
  int grid = 0;          // persistent CTAs of the GEMM passes
  int64_t ldh = 0, ldw = 0;
  int splitW = 1, splitH = 1;   // split-K factors of the two passes
  int64_t kchW = 0, kchH = 0;   // K tiles (of 32) per split
  int nG = 0, nQ = 0;           // Gram partial counts (W update CTAs, H update CTAs)
  size_t off_hcat = 0, off_wcat = 0, off_P = 0, off_S = 0, off_G = 0, off_Q = 0, off_Gred = 0, off_Qred = 0;
  size_t off_red = 0, off_Sred = 0;  // distributed all-reduce payloads (fp64)
  // fp16x2 variant (mu_tc16.cu)
  bool f16 = false;
  int64_t ldh16 = 0, ldw16 = 0;
  int splitW16 = 1, splitH16 = 1;
  int64_t kchW16 = 0, kchH16 = 0;
  size_t off_h16 = 0, off_w16 = 0, off_scales = 0;
  size_t bytes = 0;
};

struct TcMaps {
  CUtensorMap xw, xh, hcat, wcat;
  CUtensorMap xw16, xh16, hcat16, wcat16;
};

// Shapes the TC path takes: r <= 32, m, n >= 256, X 16-byte aligned with ldx % 4 == 0.
bool tc_supported(int64_t m, int64_t n, int r, int64_t ldx, const void* X);
TcPlan plan_tc(int64_t m, int64_t n, int r, int num_sms);

// Tensor maps, Hcat = [H; lo(H)] and Q partials of the initial H.
cudaError_t tc_prepare(const TcPlan& p, const float* X, int64_t ldx, float* H, char* ws, TcMaps* maps,
                       cudaStream_t st);
// Q = sum of the H-side Gram partials (fixed order)
cudaError_t tc_sum_Q(const TcPlan& p, char* ws, cudaStream_t st);
// split-K partials of P = X H^T
cudaError_t tc_pass_w(const TcPlan& p, const TcMaps& mp, char* ws, int evict_first, cudaStream_t st);
// W <- W o P / (W Q + eps); Wcat; G = W^T W (reduced)
cudaError_t tc_wupdate(const TcPlan& p, float* W, float eps, char* ws, cudaStream_t st, int it = 0);
// split-K partials of S = W^T X
cudaError_t tc_pass_h(const TcPlan& p, const TcMaps& mp, char* ws, int evict_first, cudaStream_t st);
// H <- H o S / (G H + eps); Hcat; Q partials of the new H
cudaError_t tc_hupdate(const TcPlan& p, float* H, float eps, char* ws, cudaStream_t st, int it = 0);

// explicit-operand forms (distributed path: P / S already reduced, nP = nS = 1)
cudaError_t tc_wupdate_ex(const TcPlan& p, float* W, float eps, char* ws, const double* P, int nP, const double* Q,
                          cudaStream_t st, int it = 0);
cudaError_t tc_hupdate_ex(const TcPlan& p, float* H, float eps, char* ws, const double* S, int nS, cudaStream_t st,
                          int it = 0);
// distributed payloads: ws+off_red = [P (m r) | Q (r r)], ws+off_Sred = S (n r); G (local) at ws+off_Gred
cudaError_t tc_reduce_PQ(const TcPlan& p, char* ws, cudaStream_t st);
cudaError_t tc_reduce_S(const TcPlan& p, char* ws, cudaStream_t st);

// fp16x2 variant (mu_tc16.cu): scales, fp16 operand parts and the two passes
cudaError_t tc16_prepare(const TcPlan& p, const float* X, int64_t ldx, float* H, char* ws, TcMaps* maps,
                         cudaStream_t st);
// it: iteration (-1 = the initial H of tc16_prepare); the max of the factor comes from
// the update kernel of the same iteration (parity slot), the other slot is reset
cudaError_t tc16_pack_h(const TcPlan& p, const float* H, char* ws, cudaStream_t st, int it);
cudaError_t tc16_pack_w(const TcPlan& p, const float* W, char* ws, cudaStream_t st, int it);
// BCD variants (mu_tc16.cu): max word pointer of a slot, packs that read a given slot, and
// packs that compute the max themselves (slot 7)
unsigned* tc16_max_slot(const TcPlan& p, char* ws, int slot);
cudaError_t tc16_pack_h_slot(const TcPlan& p, const float* H, char* ws, cudaStream_t st, int slot);
cudaError_t tc16_pack_w_slot(const TcPlan& p, const float* W, char* ws, cudaStream_t st, int slot);
cudaError_t tc16_pack_h_fresh(const TcPlan& p, const float* H, char* ws, cudaStream_t st);
// flush: K tiles (of 64) accumulated in fp32 in TMEM before the fp64 flush (MU: 16; BCD uses
// a shorter interval because its objective takes a difference of large terms, R25)
cudaError_t tc16_pass_w(const TcPlan& p, const TcMaps& mp, char* ws, int evict_first, cudaStream_t st,
                        int flush = 16);
cudaError_t tc16_pass_h(const TcPlan& p, const TcMaps& mp, char* ws, int evict_first, cudaStream_t st,
                        int flush = 16);

}  // namespace ntt
