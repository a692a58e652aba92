/*
 * ntt_oracle.c -- plain, slow, obviously-correct CPU oracle for the MU-NMF
 * non-negative tensor-train (nTT) sweep of arXiv 2008.01340.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the package
 * paper_2008_01340_b200/, include/, libntt.so) may include, link, load or call
 * this file.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg (and `bench.py --impl reference`) may use it.  It shares no code,
 * headers, tables or helpers with the CUDA path.
 *
 * Conventions
 *   - P:n  = /root/reference/PAPER.md line n (the paper's LaTeX), S:n = SPEC.md
 *     line n, BJ = BASELINE.json.  Readings of silent / garbled passages are
 *     the numbered list in DESIGN.md section 3 ("R1".."R19").
 *   - All arithmetic is IEEE fp64.  Input tensors may be given as fp32 (they
 *     hold exactly-representable values) or fp64; factors and every product,
 *     sum and intermediate are fp64.
 *   - Every array is row-major (C order) -- reading R8.
 *   - Loops are the definitions written out.  The only liberty taken is loop
 *     interchange that leaves each individual sum accumulated in the same
 *     sequential index order (so results do not depend on the interchange),
 *     and "#pragma omp parallel for" over INDEPENDENT outputs (each sum is still
 *     computed start-to-finish by one thread in index order), so single- and
 *     multi-threaded runs agree bit for bit.
 *
 * Parity pins (tests/test_oracle_*.py): worked 2x2 MU example (hand-derived),
 * Eckart-Young limit for r=1, rank-1 one-step closed form, Lee-Seung
 * monotonicity, fixed point, scale invariance, transpose duality, Eq. 2 brute
 * force, SPEC examples S:56-94, Eq. 4 at Fig. 1's shape.  No function here is
 * "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORA_OK 0
#define ORA_ERR_ARG 1
#define ORA_ERR_RANK 2
#define ORA_ERR_DEGENERATE 3
#define ORA_ERR_NOMEM 4

/* ------------------------------------------------------------------------ */
/* Counter-based RNG (the same TEXT spec is implemented
 * independently by the CUDA path and by ntt_inputs/).  u(seed,stream,i) is the
 * top 24 bits of a SplitMix64-finalised counter, times 2^-24, so every value
 * k*2^-24 in [0,1) is exact in fp32 and fp64.  Alg. 3 l.1 "rand",
 * BJ configs "init uniform[0,1)".                                            */
/* ------------------------------------------------------------------------ */
uint64_t ora_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

uint32_t ora_rng_u24(uint64_t seed, uint64_t stream, uint64_t i) {
    const uint64_t golden = 0x9E3779B97F4A7C15ULL;
    uint64_t key = ora_mix64(seed ^ ora_mix64(stream + golden));
    return (uint32_t)(ora_mix64(key + (i + 1ULL) * golden) >> 40);
}

double ora_rng_uniform(uint64_t seed, uint64_t stream, uint64_t i) {
    return (double)ora_rng_u24(seed, stream, i) * (1.0 / 16777216.0);
}

void ora_fill_uniform(double* out, int64_t count, uint64_t seed, uint64_t stream,
                      int64_t index_offset) {
    for (int64_t i = 0; i < count; ++i)
        out[i] = ora_rng_uniform(seed, stream, (uint64_t)(index_offset + i));
}

/* RNG stream ids (reading R20). */
uint64_t ora_stream_w(int l) { return 0x200ULL + 2ULL * (uint64_t)l; }
uint64_t ora_stream_h(int l) { return 0x201ULL + 2ULL * (uint64_t)l; }

/* ------------------------------------------------------------------------ */
/* Tensor-train helpers                                                      */
/* ------------------------------------------------------------------------ */

/* full rank vector r_0..r_d from the d-1 inner ranks; r_0 = r_d = 1. */
static void full_ranks(int d, const int32_t* inner, int64_t* r) {
    r[0] = 1;
    for (int l = 1; l < d; ++l) r[l] = inner[l - 1];
    r[d] = 1;
}

/* Packed-core offset o_l = sum_{j<l} r_{j-1} n_j r_j (cores stored back to back,
 * core l as a row-major r_{l-1} x n_l x r_l array; Table I).            */
int64_t ora_core_offset(int d, const int64_t* dims, const int32_t* inner, int l) {
    int64_t r[65];
    if (d < 1 || d > 64) return -1;
    full_ranks(d, inner, r);
    int64_t o = 0;
    for (int j = 1; j < l; ++j) o += r[j - 1] * dims[j - 1] * r[j];
    return o;
}

/* Eq. 2: A[i1..id] = sum_{k1..k_{d-1}} G1[i1,k1] G2[k1,i2,k2] ...
 * Gd[k_{d-1},id].  Written as the literal sum over every k-tuple (an odometer
 * over k_1..k_{d-1}); exponential in d -- for tiny brute-force checks only.  */
double ora_tt_element(int d, const int64_t* dims, const int32_t* inner,
                      const double* cores, const int64_t* idx) {
    int64_t r[65], o[65], k[65];
    full_ranks(d, inner, r);
    o[1] = 0;
    for (int l = 2; l <= d; ++l) o[l] = o[l - 1] + r[l - 2] * dims[l - 2] * r[l - 1];
    for (int l = 0; l <= d; ++l) k[l] = 0; /* k_0 = k_d = 0 always */
    double total = 0.0;
    for (;;) {
        double prod = 1.0;
        for (int l = 1; l <= d; ++l) {
            /* G_l[k_{l-1}, i_l, k_l] */
            int64_t e = (k[l - 1] * dims[l - 1] + idx[l - 1]) * r[l] + k[l];
            prod *= cores[o[l] + e];
        }
        total += prod;
        /* advance odometer over k_1..k_{d-1} (k_{d-1} fastest) */
        int l = d - 1;
        while (l >= 1) {
            if (++k[l] < r[l]) break;
            k[l] = 0;
            --l;
        }
        if (l < 1) break;
    }
    return total;
}

/* Eq. 1 evaluated left to right by matricised products:
 * L_1 = G_1 as n_1 x r_1; L_l = reshape(L_{l-1}, [N_{l-1}, r_{l-1}]) * G_l
 * as (N_{l-1} n_l) x r_l, where G_l is viewed as r_{l-1} x (n_l r_l).  The
 * final L_d (N x 1) is A in row-major order.  out: prod(dims) doubles.       */
int ora_tt_full(int d, const int64_t* dims, const int32_t* inner,
                const double* cores, double* out) {
    int64_t r[65];
    if (d < 1 || d > 64) return ORA_ERR_ARG;
    full_ranks(d, inner, r);
    int64_t N = dims[0];
    double* L = (double*)malloc(sizeof(double) * (size_t)(dims[0] * r[1]));
    if (!L) return ORA_ERR_NOMEM;
    memcpy(L, cores, sizeof(double) * (size_t)(dims[0] * r[1]));
    int64_t off = dims[0] * r[1];
    for (int l = 2; l <= d; ++l) {
        const int64_t nl = dims[l - 1], rp = r[l - 1], rl = r[l];
        const double* G = cores + off;
        double* Ln = (l == d) ? out : (double*)malloc(sizeof(double) * (size_t)(N * nl * rl));
        if (!Ln) { free(L); return ORA_ERR_NOMEM; }
#pragma omp parallel for schedule(static)
        for (int64_t a = 0; a < N; ++a)
            for (int64_t i = 0; i < nl; ++i)
                for (int64_t c = 0; c < rl; ++c) {
                    double s = 0.0;
                    for (int64_t k = 0; k < rp; ++k)
                        s += L[a * rp + k] * G[(k * nl + i) * rl + c];
                    Ln[(a * nl + i) * rl + c] = s;
                }
        free(L);
        L = Ln;
        N *= nl;
        off += rp * nl * rl;
    }
    if (d == 1) memcpy(out, L, sizeof(double) * (size_t)N);
    if (d == 1 || L != out) free(L);
    return ORA_OK;
}

/* Eq. 1 split at bond k (1 <= k < d): A[a, b] = sum_q L[a, q] R[q, b] with
 * L = G_1 o ... o G_k as (n_1..n_k) x r_k and R = G_{k+1} o ... o G_d as
 * r_k x (n_{k+1}..n_d), each contracted left to right by ora_tt_full on a
 * sub-train closed with an identity core.  Caller frees *L and *R.            */
static int split_LR(int d, const int64_t* dims, const int32_t* inner, const double* cores, int k,
                    double** Lout, double** Rout, int64_t* NLout, int64_t* NRout, int64_t* rkout) {
    int64_t r[65];
    full_ranks(d, inner, r);
    int64_t NL = 1, NR = 1;
    for (int l = 0; l < k; ++l) NL *= dims[l];
    for (int l = k; l < d; ++l) NR *= dims[l];
    int64_t rk = r[k];
    double* L = (double*)malloc(sizeof(double) * (size_t)(NL * rk));
    double* R = (double*)malloc(sizeof(double) * (size_t)(rk * NR));
    if (!L || !R) { free(L); free(R); return ORA_ERR_NOMEM; }
    {
        /* left sub-train: G_1..G_k followed by an identity core rk x rk x 1 */
        int64_t o_end = ora_core_offset(d, dims, inner, k + 1);
        int64_t dl[65];
        int32_t il[65];
        for (int l = 0; l < k; ++l) dl[l] = dims[l];
        dl[k] = rk;
        for (int l = 0; l < k - 1; ++l) il[l] = (int32_t)r[l + 1];
        il[k - 1] = (int32_t)rk;
        double* cl = (double*)malloc(sizeof(double) * (size_t)(o_end + rk * rk));
        if (!cl) { free(L); free(R); return ORA_ERR_NOMEM; }
        memcpy(cl, cores, sizeof(double) * (size_t)o_end);
        for (int64_t a = 0; a < rk; ++a)
            for (int64_t b = 0; b < rk; ++b) cl[o_end + a * rk + b] = (a == b) ? 1.0 : 0.0;
        int rc = ora_tt_full(k + 1, dl, il, cl, L);
        free(cl);
        if (rc) { free(L); free(R); return rc; }
    }
    {
        /* right sub-train: an identity core 1 x rk x rk followed by G_{k+1}..G_d */
        int64_t o_beg = ora_core_offset(d, dims, inner, k + 1);
        int64_t o_end = ora_core_offset(d, dims, inner, d) + r[d - 1] * dims[d - 1];
        int64_t dr[65];
        int32_t ir[65];
        dr[0] = rk;
        for (int l = k; l < d; ++l) dr[l - k + 1] = dims[l];
        for (int l = k; l < d; ++l) ir[l - k] = (int32_t)r[l];
        double* cr = (double*)malloc(sizeof(double) * (size_t)(rk * rk + (o_end - o_beg)));
        if (!cr) { free(L); free(R); return ORA_ERR_NOMEM; }
        for (int64_t a = 0; a < rk; ++a)
            for (int64_t b = 0; b < rk; ++b) cr[a * rk + b] = (a == b) ? 1.0 : 0.0;
        memcpy(cr + rk * rk, cores + o_beg, sizeof(double) * (size_t)(o_end - o_beg));
        int rc = ora_tt_full(d - k + 1, dr, ir, cr, R);
        free(cr);
        if (rc) { free(L); free(R); return rc; }
    }
    *Lout = L;
    *Rout = R;
    *NLout = NL;
    *NRout = NR;
    *rkout = rk;
    return ORA_OK;
}

/* Same contraction, rounded once to fp32 (synthetic inputs are fp32)
 * plus optional additive noise amp*u(seed, noise_stream, flat index) added in
 * fp64 before rounding (reading R12).  Split at the middle bond k = d/2.      */
int ora_tt_full_f32(int d, const int64_t* dims, const int32_t* inner,
                    const double* cores, double noise_amp, uint64_t seed,
                    uint64_t noise_stream, float* out) {
    if (d < 2 || d > 64) return ORA_ERR_ARG;
    double *L, *R;
    int64_t NL, NR, rk;
    int rc = split_LR(d, dims, inner, cores, d / 2, &L, &R, &NL, &NR, &rk);
    if (rc) return rc;
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < NL; ++a)
        for (int64_t b = 0; b < NR; ++b) {
            double s = 0.0;
            for (int64_t q = 0; q < rk; ++q) s += L[a * rk + q] * R[q * NR + b];
            int64_t flat = a * NR + b;
            if (noise_amp != 0.0) s += noise_amp * ora_rng_uniform(seed, noise_stream, (uint64_t)flat);
            out[flat] = (float)s;
        }
    free(L);
    free(R);
    return ORA_OK;
}

/* Eq. 3 of a TT against fp32 A, the reconstruction formed on the fly
 * from the bond-k split (fp64, direct differences).  Row sums of A-blocks are
 * accumulated per row a in order, rows summed in order: a fixed order.
 * Returns -1 if ||A|| = 0, -2 on allocation failure.                          */
double ora_tt_rel_error_split_f32(int d, const int64_t* dims, const int32_t* inner, const double* cores,
                                  const float* A, int k) {
    if (d < 2 || d > 64 || k < 1 || k >= d) return -3.0;
    double *L, *R;
    int64_t NL, NR, rk;
    if (split_LR(d, dims, inner, cores, k, &L, &R, &NL, &NR, &rk)) return -2.0;
    double* rn = (double*)malloc(sizeof(double) * (size_t)NL);
    double* rd = (double*)malloc(sizeof(double) * (size_t)NL);
    if (!rn || !rd) { free(L); free(R); free(rn); free(rd); return -2.0; }
#pragma omp parallel for schedule(static)
    for (int64_t a = 0; a < NL; ++a) {
        double num = 0.0, den = 0.0;
        for (int64_t b = 0; b < NR; ++b) {
            double s = 0.0;
            for (int64_t q = 0; q < rk; ++q) s += L[a * rk + q] * R[q * NR + b];
            double x = (double)A[a * NR + b], e = x - s;
            num += e * e;
            den += x * x;
        }
        rn[a] = num;
        rd[a] = den;
    }
    double num = 0.0, den = 0.0;
    for (int64_t a = 0; a < NL; ++a) { num += rn[a]; den += rd[a]; }
    free(L); free(R); free(rn); free(rd);
    if (den == 0.0) return -1.0;
    return sqrt(num) / sqrt(den);
}

/* ------------------------------------------------------------------------ */
/* MU NMF building blocks.  X is m x n (fp32 `Xf` or fp64 `Xd`, exactly one  */
/* non-NULL), W is m x r, H is r x n, all row-major.                          */
/* MU rule: Lee-Seung Frobenius, named at P:312 / P:461, rule per BJ north_star
 * and S:350 (reading R1), W first then H with the NEW W (R2), additive eps (R3),
 * evaluated as (w * num) / (den + eps) (R4).                                 */
/* ------------------------------------------------------------------------ */
#define XAT(i, j) (Xf ? (double)Xf[(int64_t)(i) * n + (j)] : Xd[(int64_t)(i) * n + (j)])

/* P = X H^T  (m x r):  P[i][k] = sum_j X[i][j] H[k][j].  Alg. 5 l.2.
 * Loop order (i outer, j middle, k inner) keeps each sum in j order.        */
void ora_xht(const float* Xf, const double* Xd, int64_t m, int64_t n, int r,
             const double* H, double* P) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i) {
        double acc[64];
        for (int k = 0; k < r; ++k) acc[k] = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            double x = XAT(i, j);
            for (int k = 0; k < r; ++k) acc[k] += x * H[(int64_t)k * n + j];
        }
        for (int k = 0; k < r; ++k) P[i * r + k] = acc[k];
    }
}

/* Q = H H^T (r x r): Q[k][l] = sum_j H[k][j] H[l][j].  Alg. 4. */
void ora_gram_rows(const double* H, int r, int64_t n, double* Q) {
#pragma omp parallel for schedule(static) collapse(2)
    for (int k = 0; k < r; ++k)
        for (int l = 0; l < r; ++l) {
            double s = 0.0;
            for (int64_t j = 0; j < n; ++j) s += H[(int64_t)k * n + j] * H[(int64_t)l * n + j];
            Q[k * r + l] = s;
        }
}

/* G = W^T W (r x r): G[k][l] = sum_i W[i][k] W[i][l].  Alg. 4. */
void ora_gram_cols(const double* W, int64_t m, int r, double* G) {
    for (int k = 0; k < r; ++k)
        for (int l = 0; l < r; ++l) {
            double s = 0.0;
            for (int64_t i = 0; i < m; ++i) s += W[i * r + k] * W[i * r + l];
            G[k * r + l] = s;
        }
}

/* W half-iteration, given P = X H^T and Q = H H^T:
 *   D[i][k] = sum_l W[i][l] Q[l][k];  W[i][k] <- (W[i][k] P[i][k]) / (D[i][k] + eps).
 * All D computed from the OLD W before any W entry changes.                 */
void ora_w_update(double* W, int64_t m, int r, const double* P, const double* Q, double eps) {
    double* D = (double*)malloc(sizeof(double) * (size_t)(m * r));
    for (int64_t i = 0; i < m; ++i)
        for (int k = 0; k < r; ++k) {
            double s = 0.0;
            for (int l = 0; l < r; ++l) s += W[i * r + l] * Q[l * r + k];
            D[i * r + k] = s;
        }
    for (int64_t i = 0; i < m; ++i)
        for (int k = 0; k < r; ++k)
            W[i * r + k] = (W[i * r + k] * P[i * r + k]) / (D[i * r + k] + eps);
    free(D);
}

/* S[:, j] = W^T X[:, j] for the columns listed in `cols` (all columns when
 * cols == NULL; then ncols must equal n).  S is r x ncols.  Alg. 6 l.2
 * (P:287): S[k][c] = sum_i W[i][k] X[i][j_c].                               */
void ora_wtx_cols(const double* W, const float* Xf, const double* Xd, int64_t m,
                  int64_t n, int r, const int64_t* cols, int64_t ncols, double* S) {
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < ncols; ++c) {
        int64_t j = cols ? cols[c] : c;
        for (int k = 0; k < r; ++k) {
            double s = 0.0;
            for (int64_t i = 0; i < m; ++i) s += W[i * r + k] * XAT(i, j);
            S[(int64_t)k * ncols + c] = s;
        }
    }
}

/* H half-iteration on the listed columns, given S = W^T X (at those columns,
 * r x ncols) and G = W^T W:
 *   E[k][j] = sum_l G[k][l] H[l][j];  H[k][j] <- (H[k][j] S[k][j]) / (E[k][j] + eps).
 * Hcols: r x ncols slice of H (in/out).                                      */
void ora_h_update_cols(double* Hcols, int64_t ncols, int r, const double* S,
                       const double* G, double eps) {
#pragma omp parallel for schedule(static)
    for (int64_t c = 0; c < ncols; ++c) {
        double E[64];
        for (int k = 0; k < r; ++k) {
            double s = 0.0;
            for (int l = 0; l < r; ++l) s += G[k * r + l] * Hcols[(int64_t)l * ncols + c];
            E[k] = s;
        }
        for (int k = 0; k < r; ++k)
            Hcols[(int64_t)k * ncols + c] =
                (Hcols[(int64_t)k * ncols + c] * S[(int64_t)k * ncols + c]) / (E[k] + eps);
    }
}

/* Objective 1/2 ||X - W H||_F^2 by direct differences (Alg. 3 l.16, P:224;
 * reading R18).                                                              */
double ora_objective(const float* Xf, const double* Xd, int64_t m, int64_t n, int r,
                     const double* W, const double* H) {
    double total = 0.0;
    for (int64_t i = 0; i < m; ++i) {
        double row = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            double wh = 0.0;
            for (int k = 0; k < r; ++k) wh += W[i * r + k] * H[(int64_t)k * n + j];
            double e = XAT(i, j) - wh;
            row += e * e;
        }
        total += row;
    }
    return 0.5 * total;
}

/* One full MU iteration (W half, then H half with the new W). */
static int mu_iteration(const float* Xf, const double* Xd, int64_t m, int64_t n, int r,
                        double eps, double* W, double* H) {
    double* P = (double*)malloc(sizeof(double) * (size_t)(m * r));
    double* S = (double*)malloc(sizeof(double) * (size_t)(r * n));
    double Q[64 * 64], G[64 * 64];
    if (!P || !S) { free(P); free(S); return ORA_ERR_NOMEM; }
    ora_xht(Xf, Xd, m, n, r, H, P);           /* P = X H^T      */
    ora_gram_rows(H, r, n, Q);                /* Q = H H^T      */
    ora_w_update(W, m, r, P, Q, eps);         /* W <- W*P/(WQ+e) */
    ora_gram_cols(W, m, r, G);                /* G = W^T W      */
    ora_wtx_cols(W, Xf, Xd, m, n, r, NULL, n, S); /* S = W^T X  */
    ora_h_update_cols(H, n, r, S, G, eps);    /* H <- H*S/(GH+e) */
    free(P);
    free(S);
    return ORA_OK;
}

/* MU NMF: `iters` iterations from the given W (m x r) and H (r x n), in place.
 * obj_trace (nullable, length iters) receives 1/2||X-WH||^2 after each
 * iteration.  Problem statement: Alg. 3 Ensure.                      */
int ora_nmf_mu(const float* Xf, const double* Xd, int64_t m, int64_t n, int r, int iters,
               double eps, double* W, double* H, double* obj_trace) {
    if ((Xf == NULL) == (Xd == NULL) || m < 1 || n < 1 || r < 1 || r > 64 || iters < 0)
        return ORA_ERR_ARG;
    for (int it = 0; it < iters; ++it) {
        int rc = mu_iteration(Xf, Xd, m, n, r, eps, W, H);
        if (rc) return rc;
        if (obj_trace) obj_trace[it] = ora_objective(Xf, Xd, m, n, r, W, H);
    }
    return ORA_OK;
}

/* ------------------------------------------------------------------------ */
/* nTT sweep with fixed ranks: Alg. 2 and section III-A
 * with the SVD rank rule replaced by the caller's ranks (reading R11).
 *   T_0 = A;  for l = 1..d-1:  X = reshape(T_{l-1}, [r_{l-1} n_l, prod_{i>l} n_i])
 *   (R9), W_l, H_l initialised from streams (R20) by GLOBAL row-major index,
 *   MU for `iters` iterations, core_l[k][i][j] = W_l[k n_l + i][j] (Alg. 2 l.8),
 *   T_l = H_l (l.9);  core_d[k][i][0] = T_{d-1}[k][i] (l.11).
 * cores: packed fp64, sum_l r_{l-1} n_l r_l entries.  The unfolding is an
 * explicit copy here (reading R8: X[i][j] = T_flat[i*n + j]).               */
/* ------------------------------------------------------------------------ */
int ora_check_ranks(int d, const int64_t* dims, const int32_t* inner) {
    if (d < 2 || d > 64) return ORA_ERR_ARG;
    for (int l = 0; l < d; ++l)
        if (dims[l] < 1) return ORA_ERR_ARG;
    int64_t r[65];
    full_ranks(d, inner, r);
    for (int l = 1; l < d; ++l) {
        int64_t rest = 1;
        for (int i = l; i < d; ++i) rest *= dims[i];
        int64_t rows = r[l - 1] * dims[l - 1];
        if (r[l] < 1 || r[l] > rows || r[l] > rest || r[l] > 64) return ORA_ERR_RANK;
    }
    return ORA_OK;
}

int ora_ntt_decompose(const float* A, int d, const int64_t* dims, const int32_t* inner,
                      int iters, uint64_t seed, double eps, double* cores) {
    int rc = ora_check_ranks(d, dims, inner);
    if (rc) return rc;
    int64_t r[65];
    full_ranks(d, inner, r);
    int64_t N = 1;
    for (int l = 0; l < d; ++l) N *= dims[l];
    const float* Tf = A; /* T_0 = A (fp32 input) */
    double* Td = NULL;   /* T_l = H_l (fp64) for l >= 1 */
    int64_t off = 0;
    int64_t rest = N;    /* prod_{i>=l} n_i */
    for (int l = 1; l <= d - 1; ++l) {
        const int64_t m = r[l - 1] * dims[l - 1];
        rest /= dims[l - 1];
        const int64_t n = rest; /* prod_{i>l} n_i */
        const int rl = (int)r[l];
        /* explicit unfold copy: X[i][j] = T_flat[i*n + j] */
        float* Xf = NULL;
        double* Xd = NULL;
        if (Tf) {
            Xf = (float*)malloc(sizeof(float) * (size_t)(m * n));
            if (!Xf) return ORA_ERR_NOMEM;
            for (int64_t i = 0; i < m; ++i)
                for (int64_t j = 0; j < n; ++j) Xf[i * n + j] = Tf[i * n + j];
        } else {
            Xd = (double*)malloc(sizeof(double) * (size_t)(m * n));
            if (!Xd) return ORA_ERR_NOMEM;
            for (int64_t i = 0; i < m; ++i)
                for (int64_t j = 0; j < n; ++j) Xd[i * n + j] = Td[i * n + j];
        }
        double* W = (double*)malloc(sizeof(double) * (size_t)(m * rl));
        double* H = (double*)malloc(sizeof(double) * (size_t)(rl * n));
        if (!W || !H) return ORA_ERR_NOMEM;
        ora_fill_uniform(W, m * rl, seed, ora_stream_w(l), 0);
        ora_fill_uniform(H, rl * n, seed, ora_stream_h(l), 0);
        rc = ora_nmf_mu(Xf, Xd, m, n, rl, iters, eps, W, H, NULL);
        if (rc) return rc;
        /* core_l[k][i][j] = W[k*n_l + i][j]: the same numbers in the same order */
        for (int64_t k = 0; k < r[l - 1]; ++k)
            for (int64_t i = 0; i < dims[l - 1]; ++i)
                for (int64_t j = 0; j < rl; ++j)
                    cores[off + (k * dims[l - 1] + i) * rl + j] = W[(k * dims[l - 1] + i) * rl + j];
        off += m * rl;
        free(W);
        free(Xf);
        free(Xd);
        free(Td);
        Td = H;
        Tf = NULL;
    }
    /* last core G_d[k][i][0] = T_{d-1}[k][i] */
    for (int64_t k = 0; k < r[d - 1]; ++k)
        for (int64_t i = 0; i < dims[d - 1]; ++i) cores[off + k * dims[d - 1] + i] = Td[k * dims[d - 1] + i];
    free(Td);
    return ORA_OK;
}

/* Eq. 3: ||A - B||_F / ||A||_F by direct differences (R18).
 * Returns -1 when ||A|| = 0 (DegenerateInput).                         */
double ora_rel_error_f32(const float* A, const double* B, int64_t N) {
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < N; ++i) {
        double a = (double)A[i], e = a - B[i];
        num += e * e;
        den += a * a;
    }
    if (den == 0.0) return -1.0;
    return sqrt(num) / sqrt(den);
}

double ora_rel_error(const double* A, const double* B, int64_t N) {
    double num = 0.0, den = 0.0;
    for (int64_t i = 0; i < N; ++i) {
        double e = A[i] - B[i];
        num += e * e;
        den += A[i] * A[i];
    }
    if (den == 0.0) return -1.0;
    return sqrt(num) / sqrt(den);
}

/* Eq. 4: C = prod n_i / sum n_i r_{i-1} r_i. */
double ora_compression_ratio(int d, const int64_t* dims, const int32_t* inner) {
    int64_t r[65];
    full_ranks(d, inner, r);
    double num = 1.0, den = 0.0;
    for (int i = 1; i <= d; ++i) {
        num *= (double)dims[i - 1];
        den += (double)dims[i - 1] * (double)r[i - 1] * (double)r[i];
    }
    return num / den;
}

/* Relative error of a TT (packed fp64 cores) against an fp32 tensor, by direct
 * differences, WITHOUT materialising the reconstruction: each element of the
 * reconstruction is formed by the left-to-right vector-matrix product of Eq. 2
 * ("sequential vector-matrix products").  Used at full sizes.           */
double ora_tt_rel_error_f32(int d, const int64_t* dims, const int32_t* inner,
                            const double* cores, const float* A) {
    int64_t r[65], o[65];
    full_ranks(d, inner, r);
    o[1] = 0;
    for (int l = 2; l <= d; ++l) o[l] = o[l - 1] + r[l - 2] * dims[l - 2] * r[l - 1];
    int64_t N = 1;
    for (int l = 0; l < d; ++l) N *= dims[l];
    /* Fixed two-level order (blocks of 2^16 elements summed sequentially, then
     * the block sums sequentially) so the result does not depend on threads. */
    const int64_t BLK = (int64_t)1 << 16;
    const int64_t nblk = (N + BLK - 1) / BLK;
    double* bnum = (double*)calloc((size_t)nblk, sizeof(double));
    double* bden = (double*)calloc((size_t)nblk, sizeof(double));
    if (!bnum || !bden) { free(bnum); free(bden); return -2.0; }
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t b = 0; b < nblk; ++b) {
      double num = 0.0, den = 0.0;
      int64_t end = (b + 1) * BLK < N ? (b + 1) * BLK : N;
      for (int64_t flat = b * BLK; flat < end; ++flat) {
        int64_t idx[64], t = flat;
        for (int l = d - 1; l >= 0; --l) { idx[l] = t % dims[l]; t /= dims[l]; }
        double v[64], w[64];
        for (int64_t c = 0; c < r[1]; ++c) v[c] = cores[o[1] + idx[0] * r[1] + c];
        for (int l = 2; l <= d; ++l) {
            for (int64_t c = 0; c < r[l]; ++c) {
                double s = 0.0;
                for (int64_t k = 0; k < r[l - 1]; ++k)
                    s += v[k] * cores[o[l] + (k * dims[l - 1] + idx[l - 1]) * r[l] + c];
                w[c] = s;
            }
            for (int64_t c = 0; c < r[l]; ++c) v[c] = w[c];
        }
        double a = (double)A[flat], e = a - v[0];
        num += e * e;
        den += a * a;
      }
      bnum[b] = num;
      bden[b] = den;
    }
    double num = 0.0, den = 0.0;
    for (int64_t b = 0; b < nblk; ++b) { num += bnum[b]; den += bden[b]; }
    free(bnum);
    free(bden);
    if (den == 0.0) return -1.0;
    return sqrt(num) / sqrt(den);
}
