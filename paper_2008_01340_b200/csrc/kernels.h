// kernels.h -- internal launcher declarations of libntt (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace ntt {

// ---- RNG -------------------------------------------------------------------
cudaError_t launch_fill_uniform(float* p, int64_t count, uint64_t seed, uint64_t stream,
                                int64_t index_offset, cudaStream_t st);

// ---- generic (2-pass) MU building blocks ------------------------------------
// Partials are fp64, laid out [split][rows*r].
struct XhtPlan {
  int ncs;          // column splits (number of partial copies)
  int nrb;          // row blocks
  int64_t chunk;    // columns per split (multiple of the tile width)
};
XhtPlan plan_xht(int64_t m, int64_t n, int num_sms);
// Ppart[b][i*r+k] = sum_{j in split b} X[i][j] * H[k][j]
cudaError_t launch_xht_partial(const float* X, int64_t ldx, int64_t m, int64_t n, const float* H,
                               int64_t ldh, int r, const XhtPlan& pl, double* Ppart, cudaStream_t st);

// W <- W o P / (W Q + eps) with P = sum_b Ppart[b], Q = sum_b Qpart[b] (fixed order);
// Gpart[c][k*r+l] = sum over CTA c's rows of Wn[i][k] Wn[i][l]  (c < wupdate_ctas(m))
int wupdate_ctas(int64_t m, int r);
cudaError_t launch_wupdate(float* W, int64_t m, int r, const double* Ppart, int nP, const double* Qpart,
                           int nQ, float eps, double* Gpart, cudaStream_t st);

// H pass: G = sum_c Gpart[c]; S = W^T X; H <- H o S / (G H + eps) in place.
// If Ppart != nullptr, also accumulates per-CTA partials of P' = X Hn^T, Q' = Hn Hn^T
// (the 1-pass fusion; requires m*r <= kMaxAccMR) into Ppart[cta], Qpart[cta].
constexpr int64_t kMaxAccMR = 4096;
// split-K H pass (no P, Q accumulation) for few column tiles and many rows: hpass_splits() splits
// (0 = not used), Spart = splits x n x Rpad fp64 (Rpad = r rounded up to 2/4/8/16/32/64)
int hpass_splits(int64_t m, int64_t n, int num_sms);
cudaError_t launch_hpass_sk(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, int r,
                            const double* Gpart, int nG, float eps, float* H, int ks, double* Spart, double* Gred,
                            cudaStream_t st);
int hpass_ctas(int64_t m, int64_t n, int r, bool acc, int num_sms);
cudaError_t launch_hpass(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, int r,
                         const double* Gpart, int nG, float eps, float* H, int grid, double* Ppart,
                         double* Qpart, cudaStream_t st);

// tiny mode (mu_tiny.cu): the whole MU loop of a small X (m n <= 48k, m <= 64,
// r <= 16) in one CTA from shared memory
bool tiny_supported(int64_t m, int64_t n, int r);
cudaError_t launch_tiny(const float* X, int64_t ldx, int64_t m, int64_t n, int r, int iters, float eps, float* W,
                        float* H, cudaStream_t st, unsigned long long* trace = nullptr);

// cluster mode (mu_cluster.cu): the whole MU loop of a mid-size X (m <= 256, r <= 16, at most
// ~16 K entries of X per CTA) in one thread-block cluster of <= 16 CTAs, X resident in the
// cluster's distributed shared memory; cluster_size_for = 0 when the shape does not fit
int cluster_size_for(int64_t m, int64_t n, int r);
bool cluster_supported(int64_t m, int64_t n, int r);
cudaError_t launch_cluster_mu(const float* X, int64_t ldx, int64_t m, int64_t n, int r, int iters, float eps, float* W,
                              float* H, cudaStream_t st, unsigned long long* trace = nullptr);



// SVD rank rule of Alg. 2 l.5-6 (tt_rank.cu): Gram of X (N = min(m, n) <= kRankMaxN) ->
// eigenvalues (Householder + bisection: one CTA for N <= 512, a cooperative grid-wide reduction
// and a warp-per-eigenvalue multisection above) -> r = smallest k with tail energy <= tt_eps.
// Writes d_rank[0] (and the N eigenvalues ascending to d_eig when non-null).
constexpr int kRankMaxN = 4096;
// the grid-wide part for N > 512 (tt_rank.cu): cooperative Householder reduction of C (destroyed;
// reflector k stored in row k of Vh when non-null) to the tridiagonal (d, e), then every
// eigenvalue ascending into lam by warp multisection.  p: N doubles scratch, ctr: 64 bytes.
cudaError_t launch_tridiag_eig(double* C, int N, double* p, double* d, double* e, double* lam, unsigned* ctr,
                               double* Vh, int num_sms, cudaStream_t st);
size_t rank_rule_bytes(int64_t N, int64_t T, int num_sms);
cudaError_t launch_rank_rule(const float* X, int64_t m, int64_t n, int64_t ldx, double tt_eps, char* ws,
                             int num_sms, int* d_rank, double* d_eig, cudaStream_t st);

// fp64 Gram of X (X X^T if m <= n else X^T X) into ws (partials, then C = *Cout, N x N);
// needs rank_rule_bytes(min(m, n), max(m, n), num_sms)
cudaError_t launch_gram(const float* X, int64_t m, int64_t n, int64_t ldx, char* ws, int num_sms, double** Cout,
                        cudaStream_t st);

// TT-SVD baseline (tt_svd.cu, SURVEY s.8(f) f4): eigenvectors of the top r eigenvalues of a
// symmetric PSD C (N <= kRankMaxN: one CTA up to 512, the grid reduction + k_svd_vec +
// k_backtransform above; r <= 64 chosen by the tail rule and capped at rcap)
size_t svd_eig_bytes(int64_t N);
cudaError_t launch_svd_eig(double* C, int N, char* ws, double tt_eps, int rcap, double* eig_asc, double* lam,
                           int* d_rank, double* U, int num_sms, cudaStream_t st);
cudaError_t launch_sign_cols(const double* M, int64_t rows, int r, const double* scale, float* out, double* sgn,
                             cudaStream_t st);
cudaError_t launch_rows_from_spart(const double* Spart, int nS, int64_t n, int r, float* Xn, cudaStream_t st);
cudaError_t launch_v_rows(const double* V, int64_t n, int r, const double* mult, const double* sgn, float* out,
                          cudaStream_t st);
cudaError_t launch_sing(const double* lam, int r, double* s, double* inv, cudaStream_t st);

// BCD NMF building blocks (bcd.cu, Alg. 3).  Device state block (doubles):
enum BcdState {
  BS_XX = 0,      // ||X||_F^2
  BS_W0 = 1,      // ||W0||_F^2
  BS_H0 = 2,      // ||H0||_F^2
  BS_LW = 3,      // L_W of this iteration (||H_prev H_prev^T||_2)
  BS_LH = 4,      // L_H of this iteration (||W^T W||_2)
  BS_OBJNEW = 5,  // objective of the candidate (W, H)
  BS_OBJ = 6,     // last accepted objective
  BS_T = 7,       // extrapolation t
  BS_LWP = 8,     // L_W, L_H of the last accepted iteration
  BS_LHP = 9,
  BS_ACC = 10,    // 1 = accepted (extrapolation), 0 = correction
  BS_WW = 11,     // extrapolation weights w_W, w_H
  BS_WH = 12,
  BS_IT = 13,     // iteration counter (trace index)
  BS_DELTA = 14,
  BS_ROLE = 15,   // one-pass path: which of (H, H_prev's buffer) holds the candidate (0 / 1)
  BS_FOLD = 16,   // one-pass path: H_m is read as a H_prev - b H_prev2 inside the pass (no H commit)
  BS_FORCE = 17,  // test hook: bit i set = the l.17 test of iteration i is treated as true
  BS_COUNT = 18
};
int bcd_w_ctas(int64_t m);
cudaError_t launch_bcd_w(const float* Wm, int64_t m, int r, const double* P, const double* Q, const double* LW,
                         float* W, double* cpart, cudaStream_t st);
cudaError_t launch_bcd_wnorm(float* W, float* Wp, int64_t m, int r, const double* c, double* Gpart, unsigned* maxw,
                             cudaStream_t st);
cudaError_t launch_bcd_hscale(double* sH, int r, const double* c, cudaStream_t st);
// role-swapped H buffers (one-pass path): B[role] holds the candidate, B[1 - role] H_prev
cudaError_t launch_bcd_commit_h_role(float* B0, float* B1, float* Hm, int r, int64_t n, const double* sH,
                                     const double* bs, cudaStream_t st);
cudaError_t launch_bcd_hout_role(float* B0, float* B1, int r, int64_t n, const double* sH, const double* bs,
                                 cudaStream_t st);
cudaError_t launch_bcd_hout(const float* Hp, int r, int64_t n, double* sH, float* out, int init, const double* bs,
                            cudaStream_t st);
// one-CTA W side / post-pass stages for small W (bcd_cta_ok: r <= 16, m * rclass <= 8192)
bool bcd_cta_ok(int64_t m, int r);
cudaError_t launch_bcd_wside(const float* Wm, float* W, float* Wp, int m, int r, const double* Pc, const double* Qc,
                             double* bs, double* c, double* G, double* sH, cudaStream_t st);
cudaError_t launch_bcd_post(const double* Ppart, int nP, const double* Qpart, int nQ, int m, int r, const float* W,
                            float* Wm, float* Wp, double* Pc, double* Qc, const double* c, const double* G, double* bs,
                            double* trace, cudaStream_t st);
cudaError_t launch_bcd_commit_h(const float* H, float* Hm, float* Hp, int r, int64_t n, const double* sH,
                                const double* bs, cudaStream_t st);
cudaError_t launch_bcd_shup(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, int r, const double* G,
                            const double* LH, const float* Hm, const double* sHm, float* H, cudaStream_t st);
int bcd_spart_splits(int64_t m, int64_t n, int num_sms);
cudaError_t launch_bcd_spart(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W, int r, int nsplit,
                             double* Spart, cudaStream_t st);
cudaError_t launch_bcd_hup(const double* Spart, int nS, int64_t n, int r, const double* G, const double* LH,
                           const float* Hm, const double* sHm, float* H, unsigned* maxh, int num_sms, cudaStream_t st);
int bcd_dot_ctas(int64_t len, int num_sms);
cudaError_t launch_bcd_psum_dot(const double* part, int nparts, int64_t len, const float* W, double* P,
                                double* dotpart, int num_sms, cudaStream_t st);
cudaError_t launch_spec_norm(const double* M, int r, double* out, cudaStream_t st);
cudaError_t launch_bcd_init(double* bs, double delta, bool fold, uint64_t force, cudaStream_t st);
cudaError_t launch_bcd_decide(double* bs, double* trace, const double* dotpart, int ndot, const double* G,
                              const double* Q, int r, unsigned* mxslots, cudaStream_t st);
cudaError_t launch_bcd_commit(const float* V, float* Vm, float* Vp, int64_t cnt, const double* bs, int widx,
                              cudaStream_t st);
cudaError_t launch_bcd_commit_pq(double* Pc, const double* Pn, int64_t m, int r, double* Qc, const double* Qn,
                                 const double* c, const double* bs, double* sH, cudaStream_t st);
cudaError_t launch_scale_copy(const float* src, float* a, float* b, int64_t cnt, const double* num, const double* den,
                              cudaStream_t st);
int sumsq_ctas();
cudaError_t launch_sumsq(const float* v, int64_t rows, int64_t cols, int64_t ld, double* part, cudaStream_t st,
                         bool evict_first = false);

// 1/2 ||X - W H||^2 partial sums (fp64), one per CTA; returns number of partials.
int objective_ctas(int64_t n);
cudaError_t launch_objective(const float* X, int64_t ldx, int64_t m, int64_t n, const float* W,
                             const float* H, int r, double* part, cudaStream_t st);

// ---- tensor-train contraction ------------------------------------------------
// out[(a*nl+i)*rl+c] = sum_k L[a*rp+k] * G[(k*nl+i)*rl+c]      (left step)
cudaError_t launch_contract_left(const float* L, int64_t N, int rp, const float* G, int64_t nl, int rl,
                                 float* out, cudaStream_t st);
// out[k*(nl*NR) + i*NR + b] = sum_c G[(k*nl+i)*rl+c] * R[c*NR+b] (right step)
cudaError_t launch_contract_right(const float* G, int rp, int64_t nl, int rl, const float* R, int64_t NR,
                                  float* out, cudaStream_t st);
// A~[a,b] = sum_q L[a*rk+q] R[q*NR+b]; optional out (+ noise), optional error partials vs ref
int stream_ctas(int64_t NL, int64_t NR, int num_sms);
cudaError_t launch_tt_stream(const float* L, const float* R, int64_t NL, int64_t NR, int rk, float* out,
                             float noise_amp, uint64_t noise_key, const float* ref, double* err_part,
                             int grid, cudaStream_t st);

}  // namespace ntt

namespace ntt {
// out[t] = sum_b part[b*len + t]   (fixed order b = 0..n-1)
cudaError_t launch_sum_partials(const double* part, int nparts, int64_t len, double* out, cudaStream_t st);
// H init for a last-mode column block (DESIGN.md s.7): H[k][c] = u(key, k*nglob + (c/b)*nd + off + c%b)
// validation pass: number of entries that are not >= 0 (negatives, NaN) into *bad (device)
cudaError_t launch_count_not_nonneg(const float* v, int64_t rows, int64_t cols, int64_t ld, unsigned long long* bad,
                                    int num_sms, cudaStream_t st);
cudaError_t launch_fill_uniform_cols(float* H, int r, int64_t nloc, int64_t b, int64_t nd, int64_t off, int64_t nglob,
                                     uint64_t seed, uint64_t stream, cudaStream_t st);
// gathered rank-major blocks [g][r][b_g] -> core [r][nd]
// fixed-order sum of npart (a, b) pairs -> out[0..1]
cudaError_t launch_sum_pairs(const double* part, int npart, double* out, cudaStream_t st);
cudaError_t launch_read_stream(const void* buf, int64_t bytes, float* sink, int num_sms, cudaStream_t st);
cudaError_t launch_gather_last_core(const float* gath, int64_t r, int64_t nd, int nranks, float* core, cudaStream_t st);
}  // namespace ntt
