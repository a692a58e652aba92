/*
 * ntt.h -- C ABI of the B200-native MU-NMF non-negative tensor-train library
 * (libntt.so), after arXiv 2008.01340 "Distributed Non-Negative Tensor Train
 * Decomposition".
 *
 * Citation keys: P:n = line n of the paper's LaTeX (/root/reference/PAPER.md at
 * build time; the library never reads it), Alg./Eq. numbers are the paper's.
 * Readings of silent or garbled passages (R1..R20) are listed in DESIGN.md s.3.
 *
 * General conventions (all entry points)
 *   - Element type is IEEE fp32, every matrix / tensor is ROW-MAJOR (C order,
 *     reading R8).  Index types are int64_t; ranks int32_t.
 *   - Pointers: unless stated otherwise a data pointer may be DEVICE memory
 *     (cudaMalloc / torch CUDA tensors, on the handle's device) or HOST memory
 *     (pageable or, for speed, pinned).  Host buffers are staged through device
 *     memory by the library inside the call (host<->device copies are part of
 *     the call).  The caller owns every buffer; the library never frees caller
 *     memory and never keeps a caller pointer after the call returns.
 *   - Work is enqueued on the handle's CUDA stream and is stream-ordered.  A call
 *     that returns a host scalar (rel_err, objective_trace, host outputs)
 *     synchronises that stream before returning.  Other calls return as soon as
 *     the work is enqueued.
 *   - Errors: every entry point validates its arguments BEFORE launching any
 *     kernel and returns a non-zero ntt_status without side effects on invalid
 *     input.  A CUDA failure after launch returns NTT_ERR_CUDA; outputs are then
 *     unspecified.  ntt_last_error(h) gives a one-line description.
 *   - A handle is bound to one device and one stream; it is not thread-safe
 *     (use one handle per host thread / per rank).
 *   - No silent CPU fallback exists: every arithmetic step runs in this
 *     library's sm_100a kernels.  Without a usable CUDA device ntt_create fails.
 */
#ifndef NTT_H_
#define NTT_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define NTT_ABI_VERSION 1

typedef enum {
    NTT_OK = 0,
    NTT_ERR_INVALID_ARG = 1,  /* null pointer, negative size, bad leading dim   */
    NTT_ERR_DIMENSION = 2,    /* d < 2, a dim < 1, size overflow        */
    NTT_ERR_RANK = 3,         /* rank outside 1..min(rows, cols), > 64  */
    NTT_ERR_DEGENERATE = 4,   /* ||A||_F = 0 in an error evaluation     */
    NTT_ERR_NONNEG = 5,       /* negative / NaN input (NTT_VALIDATE_NONNEG)     */
    NTT_ERR_WORKSPACE = 6,    /* caller workspace too small                    */
    NTT_ERR_CUDA = 7,         /* CUDA runtime / launch failure                 */
    NTT_ERR_NCCL = 8,         /* NCCL failure (distributed handles)            */
    NTT_ERR_UNSUPPORTED = 9   /* valid request this build does not implement   */
} ntt_status;

typedef struct ntt_handle_s* ntt_handle;

/* ---------------------------------------------------------------- handles --
 * ntt_create: bind a handle to CUDA `device` and `cuda_stream` (a cudaStream_t;
 * NULL = the legacy default stream).  Fails with NTT_ERR_CUDA if the device is
 * absent or is not sm_100 (B200).                                            */
ntt_status ntt_create(ntt_handle* out, int device, void* cuda_stream);
ntt_status ntt_destroy(ntt_handle h);
/* Change the stream subsequent calls enqueue on. */
ntt_status ntt_set_stream(ntt_handle h, void* cuda_stream);
const char* ntt_status_string(ntt_status s);
const char* ntt_last_error(ntt_handle h);
int ntt_abi_version(void);
/* Input validation (SURVEY s.8(b); SPEC's NonnegativityError).  With
 * NTT_VALIDATE_NONNEG set, ntt_nmf_mu, ntt_nmf_bcd, ntt_decompose,
 * ntt_decompose_eps and ntt_decompose_bcd first count the entries of X / A
 * that are not >= 0 (negative values or NaN) in one extra read of the input and
 * return NTT_ERR_NONNEG (nothing else launched) if there are any; the call
 * synchronises the stream for the count.  Off by default (NMF's problem
 * statement, Alg. 3 "Require X in R_+", makes it the caller's contract).
 * ntt_tt_svd never checks (the TT-SVD baseline takes any sign).  Unknown flag
 * bits give NTT_ERR_INVALID_ARG.                                             */
#define NTT_VALIDATE_NONNEG 1
ntt_status ntt_set_validation(ntt_handle h, int flags);

/* Number of kernel launches this handle has issued since creation (for the
 * bench's gpu_launches count; graph-replayed kernels are counted per replay). */
int64_t ntt_launch_count(ntt_handle h);

/* ------------------------------------------------------------- RNG / init --
 * Counter-based uniform draws (DESIGN.md s.4; Alg. 3 l.1 "rand"):
 *   p[i] = u(seed, stream, index_offset + i),  i < count,
 *   u(s, t, k) = (mix64(mix64(s ^ mix64(t + G)) + (k + 1) G) >> 40) * 2^-24,
 *   mix64 = SplitMix64 finaliser, G = 0x9E3779B97F4A7C15 (all mod 2^64).
 * Values are k * 2^-24 in [0, 1), exact in fp32.  p: device or host, count
 * floats.  Stream ids used by ntt_decompose: W init at step l = 0x200 + 2l,
 * H init = 0x201 + 2l (l = 1..d-1), indices = global row-major element index. */
ntt_status ntt_fill_uniform(ntt_handle h, float* p, int64_t count, uint64_t seed,
                            uint64_t stream, int64_t index_offset);

/* ------------------------------------------------------------------ MU NMF --
 * Multiplicative-update NMF, X ~= W H with W >= 0 (m x r), H >= 0 (r x n)
 * minimising ||X - W H||_F^2 (Alg. 3 Ensure; MU named at P:312/P:461;
 * rule per reading R1-R4):   for it = 1..iters
 *     W <- W o (X H^T) / (W (H H^T) + eps)            (Alg. 5 / Alg. 4 products)
 *     H <- H o (W^T X) / ((W^T W) H + eps)            (Alg. 6 / Alg. 4 products)
 * W is updated first and the H update uses the new W (R2).  The quotient is
 * evaluated as (w * num) / (den + eps) (R4).  eps >= 0 (the reference value is
 * 1e-16, R3).
 *   X   : m x n, row stride ldx >= n (floats), read-only.  For the fast 1-pass
 *         path X and ldx should be 16-byte aligned (ldx % 4 == 0); other inputs
 *         take a slower path, results are the same up to rounding.
 *   W,H : in/out.  On entry the initial factors (caller-drawn, e.g. with
 *         ntt_fill_uniform), on exit the factors after `iters` iterations.
 *   objective_trace : nullable HOST array of `iters` doubles; if given,
 *         receives 1/2 ||X - W H||_F^2 after each iteration (direct differences,
 *         fp64 sums; diagnostic, costs one extra pass over X per iteration).
 * Returns NTT_ERR_INVALID_ARG (null / m,n < 1 / ldx < n / iters < 0 / eps < 0)
 * or NTT_ERR_RANK (r < 1, r > min(m, n), r > 64).                            */
ntt_status ntt_nmf_mu(ntt_handle h, const float* X, int64_t m, int64_t n, int64_t ldx,
                      int32_t r, int32_t iters, float eps, float* W, float* H,
                      double* objective_trace);

/* ------------------------------------------------------------ nTT sweep ----
 * Non-negative tensor train with FIXED ranks (Alg. 2, section III-A
 * P:194, with the SVD rank rule l.5-6 replaced by the caller's ranks, R11):
 *   T_0 = A;  for l = 1..d-1:
 *     X_l = reshape(T_{l-1}, [r_{l-1} n_l, prod_{i>l} n_i])   (zero-copy, R9)
 *     W_l, H_l initialised by ntt_fill_uniform(seed, 0x200+2l / 0x201+2l)
 *     (W_l, H_l) = ntt_nmf_mu(X_l, r_l, iters, eps)
 *     core_l = reshape(W_l, [r_{l-1}, n_l, r_l])               (Alg. 2 l.8)
 *     T_l = H_l                                                (Alg. 2 l.9)
 *   core_d = reshape(T_{d-1}, [r_{d-1}, n_d, 1])               (Alg. 2 l.11)
 *   A     : prod(dims) floats, row-major n_1 x ... x n_d, entries >= 0.
 *   dims  : d extents (host).  ranks: the d-1 inner ranks r_1..r_{d-1} (host);
 *           r_0 = r_d = 1.  Valid iff 1 <= r_l <= min(r_{l-1} n_l, prod_{i>l} n_i)
 *           and r_l <= 64 (else NTT_ERR_RANK); d in [2, 64] and every dim >= 1
 *           (else NTT_ERR_DIMENSION).
 *   cores : packed output, sum_l r_{l-1} n_l r_l floats; core l (row-major
 *           r_{l-1} x n_l x r_l) starts at o_l = sum_{j<l} r_{j-1} n_j r_j.
 *   rel_err : nullable HOST double; if given, receives Eq. 3 of the
 *           resulting train against A, ||A - A~||_F / ||A||_F (as ntt_reconstruct
 *           computes it, fp64 sums), reusing the device copy of A.
 *   workspace : device scratch of >= ntt_decompose_workspace_bytes(...) bytes,
 *           or NULL to let the handle allocate (and keep) its own.          */
size_t ntt_decompose_workspace_bytes(int32_t d, const int64_t* dims, const int32_t* ranks);
ntt_status ntt_decompose(ntt_handle h, const float* A, int32_t d, const int64_t* dims,
                         const int32_t* ranks, int32_t iters, uint64_t seed, float eps,
                         float* cores, double* rel_err, void* workspace, size_t workspace_bytes);

/* ------------------------------------------- eps-driven nTT (SVD rank rule) --
 * Alg. 2 with the rank rule of l.5-6 (section III-A): at every
 * step the rank is r_l = the smallest k in [1, N], N = min(m, n) of the current
 * unfolding X_l, with sqrt(s_{k+1}^2 + ... + s_N^2) / sqrt(s_1^2 + ... + s_N^2)
 * <= tt_eps, capped at max_ranks[l-1] (nullable; default and hard limit 64); then
 * MU NMF with that rank as in ntt_decompose (same inits, eps, iters).  The squared
 * singular values are the eigenvalues of the fp64 Gram matrix of X_l (computed on
 * the device: split-K Gram, Householder tridiagonalisation and bisection), so the
 * rule is exact for tt_eps >= ~1e-7 (reading R21); each step needs
 * min(m, n) <= 4096 (else NTT_ERR_UNSUPPORTED).  The call synchronises once per step
 * (the next step's shapes depend on the chosen rank).
 *   cores : packed output (device or host) with room for cores_capacity floats;
 *           the layout is ntt_decompose's for the chosen ranks (NTT_ERR_WORKSPACE if
 *           the capacity is too small -- ranks_out is filled either way).
 *   ranks_out : d-1 chosen inner ranks (host).  rel_err: nullable, Eq. 3.
 * Single-GPU handles only (NTT_ERR_UNSUPPORTED on a distributed handle).      */
ntt_status ntt_decompose_eps(ntt_handle h, const float* A, int32_t d, const int64_t* dims, double tt_eps,
                             const int32_t* max_ranks, int32_t iters, uint64_t seed, float eps, float* cores,
                             int64_t cores_capacity, int32_t* ranks_out, double* rel_err);
/* The rank rule alone on a device matrix X (m x n, row stride ldx,
 * min(m, n) <= 4096, else NTT_ERR_UNSUPPORTED): *rank = r for tt_eps; eig
 * (nullable host, min(m, n) doubles) receives the squared singular values in
 * ascending order.  Up to 512 the eigensolver runs in one CTA; above, the
 * Householder reduction runs on the whole grid (one cooperative launch, fp64
 * matrix of min(m, n)^2 doubles in the handle's workspace).                    */
ntt_status ntt_rank_rule(ntt_handle h, const float* X, int64_t m, int64_t n, int64_t ldx, double tt_eps,
                         int32_t* rank, double* eig);

/* nTT with the BCD NMF at every step (Alg. 2 with Alg. 3 as its NMF):
 * fixed ranks (<= 32), W_l, H_l initialised as ntt_decompose (R20), `iters` BCD
 * iterations per step (R22-R27, delta as ntt_nmf_bcd), core l = the last accepted
 * W_l, next unfolding = the last accepted H_l.  A and cores: device or host;
 * layouts, rel_err and errors as ntt_decompose.  Single-GPU handles.          */
ntt_status ntt_decompose_bcd(ntt_handle h, const float* A, int32_t d, const int64_t* dims, const int32_t* ranks,
                             int32_t iters, uint64_t seed, double delta, float* cores, double* rel_err);

/* ------------------------------------------------------------ TT-SVD baseline
 * The unconstrained TT the paper compares nTT against (TT-SVD, P:78, P:88,
 * P:453; SURVEY s.8(f) f4; reading R28): the same sweep and the same rank rule
 * as ntt_decompose_eps (Alg. 2 l.4-6), with the NMF of each step replaced by the
 * truncated SVD of X_l: core l = U_r (left singular vectors, signs fixed so the
 * largest-magnitude entry of every column is positive), X_{l+1} = reshape(S_r V_r^T).
 * Singular vectors come from the fp64 Gram of the smaller side (Householder +
 * bisection + inverse iteration + Rayleigh-Ritz; one CTA up to min(m, n) = 512, the
 * Householder reduction and bisection on the whole grid above), so min(m, n) <= 4096
 * per step (else NTT_ERR_UNSUPPORTED) and ranks <= 64 (max_ranks caps further).
 * Cores may be negative.  Arguments, layouts and errors as ntt_decompose_eps.   */
ntt_status ntt_tt_svd(ntt_handle h, const float* A, int32_t d, const int64_t* dims, double tt_eps,
                      const int32_t* max_ranks, float* cores, int64_t cores_capacity, int32_t* ranks_out,
                      double* rel_err);

/* --------------------------------------------------------------- BCD NMF
 * The paper's alternative NMF (Alg. 3, distBCDnmf, P:196-240, P:254, P:294;
 * SURVEY s.8(f) f1) with readings R22-R27 (DESIGN.md s.3): prox-linear block
 * steps W = max(0, W_m - (W_m Q - P)/L_W), H = max(0, H_m - (G H_m - W^T X)/L_H)
 * with L = spectral norm of the r x r Gram (Q = H H^T, G = W^T W), column L1
 * normalisation of W compensated into H, Nesterov extrapolation with weights
 * min((t-1)/t+, delta sqrt(L_prev/L)), and a correction (return to the last
 * accepted iterates, t = 1) whenever the objective 1/2 ||X - W H||_F^2 (Gram
 * identity, fp64 sums) does not decrease.
 *   X : DEVICE, m x n row-major, row stride ldx >= n.
 *   W : DEVICE, m x r (in: W0, out: last accepted W).  H: DEVICE, r x n (in/out).
 *       W0 and H0 are rescaled to Frobenius norm sqrt(||X||_F) first (R22).
 *   delta in [0, 1) (paper: 0.9999).  objective_trace: nullable HOST, iters
 *   doubles: the accepted objective after every iteration.
 * Single-GPU handles, 1 <= r <= min(m, n, 32) (else NTT_ERR_RANK);
 * NTT_ERR_DEGENERATE if ||X||_F = 0.  One host synchronisation per iteration. */
ntt_status ntt_nmf_bcd(ntt_handle h, const float* X, int64_t m, int64_t n, int64_t ldx, int32_t r, int32_t iters,
                       double delta, float* W, float* H, double* objective_trace);

/* --------------------------------------------------- reconstruction / error
 * Contract a TT (Eq. 1):  A~ = G_1 o G_2 o ... o G_d, and/or the
 * relative error of Eq. 3: ||ref - A~||_F / ||ref||_F by direct
 * differences with fp64 sums (never the Gram identity, R18).
 *   cores : packed as in ntt_decompose.  out: nullable, prod(dims) floats.
 *   ref   : nullable, prod(dims) floats.  rel_err: nullable HOST double; needs
 *           ref.  NTT_ERR_DEGENERATE if ||ref||_F = 0.                       */
ntt_status ntt_reconstruct(ntt_handle h, int32_t d, const int64_t* dims, const int32_t* ranks,
                           const float* cores, float* out, const float* ref, double* rel_err);

/* Synthetic data (section IV-A): out = fp32(A~ + noise_amp *
 * u(seed, noise_stream, flat index)) with A~ the contraction of `cores`,
 * accumulated in fp32 along the middle bond (reading R12).  out: prod(dims). */
ntt_status ntt_generate(ntt_handle h, int32_t d, const int64_t* dims, const int32_t* ranks,
                        const float* cores, float noise_amp, uint64_t seed,
                        uint64_t noise_stream, float* out);

/* Eq. 4: C = prod n_i / sum n_i r_{i-1} r_i.  Host-only; returns a
 * negative value for invalid input.                                          */
double ntt_compression_ratio(int32_t d, const int64_t* dims, const int32_t* ranks);

/* ------------------------------------------------------------ profiling ----
 * Per-kernel-class timing for the roofline report.  When enabled, the library
 * brackets every launch of its kernels with CUDA events on the handle's stream
 * and records the launch's ALGORITHMIC bytes (DESIGN.md s.8).  ntt_profile_get
 * synchronises the stream and returns, for kernel class `cls`, the number of
 * launches, their summed device time in ms and summed algorithmic bytes.
 * Classes: 0 = fused 1-pass X-stream kernel (H update + next X H^T, H H^T),
 * 1 = X H^T pass (incl. the 1-pass prologue), 2 = W update, 3 = TT contraction
 * stream (error / generate), 4 = other, 5 = generic 2-pass H pass, 6 = tensor-core
 * X H^T pass, 7 = tensor-core W^T X pass (mu_tc.cu, tall / square X).
 * Enabling resets the counters.                                              */
/* Read-only HBM streaming ceiling ("report HBM % against ... a
 * harness-measured read-only streaming ceiling"; SURVEY s.8(d)).  Reads `bytes`
 * (> 0, multiple of 16) of the DEVICE buffer `buf` (16-byte aligned, contents
 * irrelevant, not modified; the caller owns it) once untimed and then `reps` (>= 1)
 * times with 128-bit evict-first loads from a grid of 8 x SM-count CTAs, timed with
 * CUDA events on the handle's stream, and stores bytes * reps / time in GB/s into
 * *gbps.  Synchronises the stream.  NTT_ERR_INVALID_ARG for bad sizes, alignment
 * or a non-device buffer.  A measurement utility, not part of the method.      */
ntt_status ntt_stream_ceiling(ntt_handle h, const void* buf, int64_t bytes, int32_t reps, double* gbps);

#define NTT_PROF_CLASSES 8
ntt_status ntt_profile_enable(ntt_handle h, int enable);
ntt_status ntt_profile_get(ntt_handle h, int cls, int64_t* launches, double* total_ms,
                           double* total_bytes);
/* Same, restricted to the launches issued for TT step `step` of ntt_decompose
 * (1..d-1; d = last-core gather and error pass; 0 = outside ntt_decompose;
 * -1 = all).                                                                 */
ntt_status ntt_profile_get_step(ntt_handle h, int cls, int step, int64_t* launches,
                                double* total_ms, double* total_bytes);

/* Diagnostics: with NTT_PERSIST_TRACE set when the handle is created, the
 * persistent fused MU kernel records, per pass p, 4 globaltimer stamps of CTA 0
 * (pass start, partials written, after barrier 1, after barrier 2) at
 * [4p .. 4p+3] of the returned host-readable array (4096 passes max; pass 0 is
 * the prologue), and for pass 1 of every CTA c < 1024 its start at [17408 + c]
 * and end at [16384 + c].  NULL otherwise.  Synchronises the handle's stream. */
const unsigned long long* ntt_debug_persist_trace(ntt_handle h);

/* Overlap the next input's host-to-device copy with device work already enqueued (a stream of
 * decompositions, e.g. the bench's end-to-end loop): an asynchronous copy of `count` floats
 * from host memory `src` (pinned for the copy to be asynchronous) into the next of two device
 * input slots of the handle, on an internal copy stream.  A later ntt_decompose call on this
 * handle whose A is that same host pointer with the same local element count waits for the copy
 * and reads the slot instead of copying A itself; each slot is refilled only after the last
 * decomposition that read it has finished.  The caller keeps `src` alive and unmodified until
 * that decomposition is enqueued.  Returns NTT_ERR_INVALID_ARG for a device pointer or
 * count < 1.  Allocates the slot on first use (synchronising the handle's streams).          */
ntt_status ntt_prefetch_input(ntt_handle h, const float* src, int64_t count);

/* Which kernel path ntt_nmf_mu takes for an m x n X at rank r on this handle
 * (16-byte aligned X and H, ldx = n; DESIGN.md s.6 "plan_mu"): 1 tiny (one CTA,
 * mu_tiny.cu), 2 cluster (one thread-block cluster, X in distributed shared
 * memory, mu_cluster.cu), 3 persistent one-pass (mu_fused.cu), 4 per-pass
 * one-pass, 5 tensor-core two-pass (mu_tc16.cu), 6 generic two-pass.  Lets
 * tests prove which path a parity case ran.  -1 for a null handle or r < 1. */
int32_t ntt_debug_mu_path(ntt_handle h, int64_t m, int64_t n, int32_t r);

/* Number of NCCL calls this handle has enqueued (collectives and group
 * brackets; a captured graph's calls are counted once, at capture).  Proves in
 * tests that a distributed branch ran.  -1 for a null handle.               */
int64_t ntt_collective_count(ntt_handle h);

/* Cross-GPU reduction of the MU passes on an ntt_create_dist* handle (SURVEY
 * s.8(e); the all_reduce of Alg. 4 P:256-266 on the TT partition, DESIGN.md s.7).
 *   mode 1 (default): the persistent one-pass kernels keep running for the whole
 *     MU loop of a step; after each pass CTA 0 stores this GPU's reduced fp64
 *     (X H^T, H H^T) vector (m r + r^2 <= 4352 doubles) into every rank's
 *     exchange buffer over NVLink (buffers allocated by ntt_create_dist*,
 *     exported / mapped with CUDA IPC, so all ranks must be one node's GPUs),
 *     raises a release flag there, waits for all ranks' flags, and every CTA
 *     sums the ranks' vectors in rank order -- no host round trip, no NCCL call
 *     per pass.  Shapes outside the persistent kernels use mode 0's path.
 *   mode 0: one ncclAllReduce per pass between per-pass kernel launches.
 * Both give the same sums up to the rank-order vs NCCL reduction order.
 * NTT_ERR_INVALID_ARG for other modes / non-distributed handles,
 * NTT_ERR_UNSUPPORTED for mode 1 if the buffers could not be mapped.
 * Synchronises the handle's stream.                                         */
ntt_status ntt_set_dist_exchange(ntt_handle h, int mode);

/* Number of in-kernel exchanges (passes) completed on this handle's exchange
 * buffer: a device-side counter the persistent kernels advance, read after a
 * stream synchronisation.  -1 if the handle has no exchange buffer.          */
int64_t ntt_peer_exchange_count(ntt_handle h);

/* Kernel-level diagnostics of the TT-mode partition (DESIGN.md s.7), so the
 * layouts of p > 1 ranks can be checked on one GPU:
 *  - ntt_debug_fill_uniform_cols: the local r x nloc H init of a rank that owns
 *    last-mode slices [off, off + b) of nd: local column c is global column
 *    (c / b) * nd + off + c % b, H[k][c] = u(seed, stream, k * nglob + that);
 *  - ntt_debug_gather_last_core: core[k][i] (r x nd) from the rank-major staging
 *    gath = [rank g: r x b_g block], b_g = floor((g+1) nd / p) - floor(g nd / p).
 * Device pointers; enqueued on the handle's stream.                          */
ntt_status ntt_debug_fill_uniform_cols(ntt_handle h, float* H, int32_t r, int64_t nloc, int64_t b, int64_t nd,
                                       int64_t off, int64_t nglob, uint64_t seed, uint64_t stream);
ntt_status ntt_debug_gather_last_core(ntt_handle h, const float* gath, int64_t r, int64_t nd, int32_t nranks,
                                      float* core);

/* Test hook for Alg. 3's correction branch (l.17-20): in every
 * later ntt_nmf_bcd / ntt_decompose_bcd NMF on this handle, iteration i (0-based,
 * i < 52) with bit i of `mask` set takes the correction branch whatever its
 * objective (a constructed overshoot; the oracle's `force_correct`).  0 (the
 * default) turns it off.  NTT_ERR_INVALID_ARG for a null handle.              */
ntt_status ntt_debug_bcd_force_correct(ntt_handle h, uint64_t mask);

/* ----------------------------------------------------- multi-GPU (NCCL) ----
 * One process per GPU.  Rank 0 calls ntt_get_unique_id and broadcasts the 128
 * bytes (e.g. over a torch process group); every rank then calls
 * ntt_create_dist with the same id.  Distributed layout for ntt_decompose
 * (DESIGN.md s.7): the LAST tensor mode is block-partitioned, rank g holds
 * A[..., i_d in [b_g, b_{g+1})] as a row-major n_1 x ... x n_{d-1} x (b_{g+1}-b_g)
 * tensor with b_g = floor(g n_d / p); every unfolding is then a column
 * partition, reshapes stay local, and each MU pass needs one all-reduce of the
 * fp64 (X H^T, H H^T) partials (Alg. 4/5 reduced to AR).  Cores are returned
 * replicated on every rank.  Returns NTT_ERR_UNSUPPORTED if NCCL cannot be
 * loaded.                                                                    */
ntt_status ntt_get_unique_id(void* id128);
ntt_status ntt_create_dist(ntt_handle* out, int device, void* cuda_stream, const void* id128,
                           int nranks, int rank);
/* 2-D pr x pc process grid for the plain NMF (Alg. 5 / Alg. 6, P:268-292;
 * SURVEY s.8(e)): rank = ga * pc + gb.  ntt_nmf_mu on such a handle takes the
 * LOCAL blocks: X = X[rows of block ga, columns of block gb] (m x n are the
 * local extents, blocks from ntt_dist_block over pr resp. pc parts), W = the
 * m x r rows of block ga (replicated over grid row ga), H = the r x n columns of
 * block gb (replicated over grid column gb).  Per iteration: all-reduce of
 * (X H^T, H H^T) over the grid row, of W^T W and of the W^T X block over the grid
 * column (fp64 payloads).  X never moves.  pr > 1 needs the tensor-core path
 * (r <= 32, m, n >= 256, 16-byte aligned X) else NTT_ERR_UNSUPPORTED.
 * ntt_create_dist(.., nranks, rank) == ntt_create_dist_grid(.., 1, nranks).  */
ntt_status ntt_create_dist_grid(ntt_handle* out, int device, void* cuda_stream, const void* id128,
                                int nranks, int rank, int pr, int pc);
/* grid shape and this rank's position; returns 0 (or -1 for a null handle) */
int ntt_dist_grid(ntt_handle h, int* pr, int* pc, int* ga, int* gb);
int ntt_dist_rank(ntt_handle h);
int ntt_dist_size(ntt_handle h);
/* Local extent of the last mode on `rank` for a global extent n_d over p ranks. */
int64_t ntt_dist_block(int64_t n_last, int nranks, int rank, int64_t* offset);

#ifdef __cplusplus
}
#endif
#endif /* NTT_H_ */
