"""CPU oracle for the MU-NMF nTT hot path of arXiv 2008.01340.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` leg / ``--impl reference`` arm may import this
package.  The product (``paper_2008_01340_b200``) never imports it, and the two
share no code: the arithmetic lives in ``oracle/ntt_oracle.c`` (plain C, fp64),
this module only marshals numpy arrays through ctypes.

Every function cites the passage it follows (P:n = PAPER.md line n, S:n =
SPEC.md line n); readings R1..R20 are listed in DESIGN.md section 3.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "ntt_oracle.c")
_LIB = os.path.join(_HERE, "libntt_oracle.so")

# plain C, fp64, no fast-math, no FMA contraction: the sums are the definitions.
CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11"]


def build(force: bool = False) -> str:
    """Compile oracle/ntt_oracle.c -> oracle/libntt_oracle.so (gcc)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None

_d = ctypes.c_double
_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_u64 = ctypes.c_uint64


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        sig = {
            "ora_mix64": (_u64, [_u64]),
            "ora_rng_u24": (ctypes.c_uint32, [_u64, _u64, _u64]),
            "ora_rng_uniform": (_d, [_u64, _u64, _u64]),
            "ora_fill_uniform": (None, [_p, _i64, _u64, _u64, _i64]),
            "ora_stream_w": (_u64, [ctypes.c_int]),
            "ora_stream_h": (_u64, [ctypes.c_int]),
            "ora_core_offset": (_i64, [ctypes.c_int, _p, _p, ctypes.c_int]),
            "ora_tt_element": (_d, [ctypes.c_int, _p, _p, _p, _p]),
            "ora_tt_full": (ctypes.c_int, [ctypes.c_int, _p, _p, _p, _p]),
            "ora_tt_full_f32": (ctypes.c_int, [ctypes.c_int, _p, _p, _p, _d, _u64, _u64, _p]),
            "ora_xht": (None, [_p, _p, _i64, _i64, ctypes.c_int, _p, _p]),
            "ora_gram_rows": (None, [_p, ctypes.c_int, _i64, _p]),
            "ora_gram_cols": (None, [_p, _i64, ctypes.c_int, _p]),
            "ora_w_update": (None, [_p, _i64, ctypes.c_int, _p, _p, _d]),
            "ora_wtx_cols": (None, [_p, _p, _p, _i64, _i64, ctypes.c_int, _p, _i64, _p]),
            "ora_h_update_cols": (None, [_p, _i64, ctypes.c_int, _p, _p, _d]),
            "ora_objective": (_d, [_p, _p, _i64, _i64, ctypes.c_int, _p, _p]),
            "ora_nmf_mu": (ctypes.c_int, [_p, _p, _i64, _i64, ctypes.c_int, ctypes.c_int, _d, _p, _p, _p]),
            "ora_check_ranks": (ctypes.c_int, [ctypes.c_int, _p, _p]),
            "ora_ntt_decompose": (ctypes.c_int, [_p, ctypes.c_int, _p, _p, ctypes.c_int, _u64, _d, _p]),
            "ora_rel_error_f32": (_d, [_p, _p, _i64]),
            "ora_rel_error": (_d, [_p, _p, _i64]),
            "ora_compression_ratio": (_d, [ctypes.c_int, _p, _p]),
            "ora_tt_rel_error_f32": (_d, [ctypes.c_int, _p, _p, _p, _p]),
            "ora_tt_rel_error_split_f32": (_d, [ctypes.c_int, _p, _p, _p, _p, ctypes.c_int]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


class OracleError(RuntimeError):
    pass


_ERR = {1: "invalid argument", 2: "rank error", 3: "degenerate input", 4: "out of memory"}


def _check(rc: int) -> None:
    if rc != 0:
        raise OracleError(f"oracle error {rc}: {_ERR.get(rc, '?')}")


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _dims(dims: Sequence[int]) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(dims, dtype=np.int64))


def _ranks(ranks: Sequence[int]) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(ranks, dtype=np.int32))


def _xargs(X: np.ndarray):
    X = np.ascontiguousarray(X)
    if X.dtype == np.float32:
        return X, _ptr(X), None
    X = np.ascontiguousarray(X, dtype=np.float64)
    return X, None, _ptr(X)


# ---------------------------------------------------------------- RNG ------
STREAM_NOISE = 0x300
STREAM_W0 = 0x400
STREAM_H0 = 0x401


def stream_w(l: int) -> int:
    """RNG stream of the W init at TT step l (reading R20)."""
    return int(lib().ora_stream_w(l))


def stream_h(l: int) -> int:
    """RNG stream of the H init at TT step l (reading R20)."""
    return int(lib().ora_stream_h(l))


def mix64(z: int) -> int:
    """SplitMix64 finaliser (the RNG spec's mixing function)."""
    return int(lib().ora_mix64(z))


def rng_u24(seed: int, stream: int, i: int) -> int:
    return int(lib().ora_rng_u24(seed, stream, i))


def fill_uniform(count: int, seed: int, stream: int, index_offset: int = 0) -> np.ndarray:
    """u(seed, stream, offset+i), i < count, as fp64 (values k*2^-24, exact in fp32)."""
    out = np.empty(count, dtype=np.float64)
    lib().ora_fill_uniform(_ptr(out), count, seed, stream, index_offset)
    return out


# ------------------------------------------------------------ TT algebra --
def core_offset(dims, ranks, l: int) -> int:
    D, R = _dims(dims), _ranks(ranks)
    return int(lib().ora_core_offset(len(D), _ptr(D), _ptr(R), l))


def cores_size(dims, ranks) -> int:
    full = [1, *ranks, 1]
    return int(sum(full[l] * dims[l] * full[l + 1] for l in range(len(dims))))


def tt_element(dims, ranks, cores: np.ndarray, idx) -> float:
    """Eq. 2: literal sum over every k-tuple."""
    D, R = _dims(dims), _ranks(ranks)
    C = np.ascontiguousarray(cores, dtype=np.float64)
    I = _dims(idx)
    return float(lib().ora_tt_element(len(D), _ptr(D), _ptr(R), _ptr(C), _ptr(I)))


def tt_full(dims, ranks, cores: np.ndarray) -> np.ndarray:
    """Eq. 1, left to right; returns the fp64 tensor, shape dims."""
    D, R = _dims(dims), _ranks(ranks)
    C = np.ascontiguousarray(cores, dtype=np.float64)
    out = np.empty(int(np.prod(D)), dtype=np.float64)
    _check(lib().ora_tt_full(len(D), _ptr(D), _ptr(R), _ptr(C), _ptr(out)))
    return out.reshape(tuple(int(x) for x in D))


def tt_full_f32(dims, ranks, cores: np.ndarray, noise_amp: float = 0.0, seed: int = 0,
                noise_stream: int = STREAM_NOISE) -> np.ndarray:
    """Synthetic fp32 tensor: the TT contraction (Eq. 1) split at the
    middle bond, plus noise_amp * u(seed, noise_stream, flat) (reading R12),
    accumulated in fp64 and rounded once to fp32."""
    D, R = _dims(dims), _ranks(ranks)
    C = np.ascontiguousarray(cores, dtype=np.float64)
    out = np.empty(int(np.prod(D)), dtype=np.float32)
    _check(lib().ora_tt_full_f32(len(D), _ptr(D), _ptr(R), _ptr(C), float(noise_amp), seed,
                                 noise_stream, _ptr(out)))
    return out.reshape(tuple(int(x) for x in D))


# --------------------------------------------------------- MU building blocks
def xht(X: np.ndarray, H: np.ndarray) -> np.ndarray:
    """P = X H^T (Alg. 5 l.2)."""
    X, xf, xd = _xargs(X)
    m, n = X.shape
    H = np.ascontiguousarray(H, dtype=np.float64)
    r = H.shape[0]
    P = np.empty((m, r))
    lib().ora_xht(xf, xd, m, n, r, _ptr(H), _ptr(P))
    return P


def gram_rows(H: np.ndarray) -> np.ndarray:
    """Q = H H^T (Alg. 4)."""
    H = np.ascontiguousarray(H, dtype=np.float64)
    r, n = H.shape
    Q = np.empty((r, r))
    lib().ora_gram_rows(_ptr(H), r, n, _ptr(Q))
    return Q


def gram_cols(W: np.ndarray) -> np.ndarray:
    """G = W^T W (Alg. 4)."""
    W = np.ascontiguousarray(W, dtype=np.float64)
    m, r = W.shape
    G = np.empty((r, r))
    lib().ora_gram_cols(_ptr(W), m, r, _ptr(G))
    return G


def w_update(W: np.ndarray, P: np.ndarray, Q: np.ndarray, eps: float = 1e-16) -> np.ndarray:
    """W <- W*P / (W Q + eps) (MU, reading R1-R4).  Returns a new array."""
    W = np.array(W, dtype=np.float64, order="C", copy=True)
    m, r = W.shape
    P = np.ascontiguousarray(P, dtype=np.float64)
    Q = np.ascontiguousarray(Q, dtype=np.float64)
    lib().ora_w_update(_ptr(W), m, r, _ptr(P), _ptr(Q), eps)
    return W


def wtx_cols(W: np.ndarray, X: np.ndarray, cols: Optional[Sequence[int]] = None) -> np.ndarray:
    """S = W^T X at the listed columns (Alg. 6 l.2)."""
    X, xf, xd = _xargs(X)
    m, n = X.shape
    W = np.ascontiguousarray(W, dtype=np.float64)
    r = W.shape[1]
    if cols is None:
        C, nc = None, n
    else:
        C = _dims(cols)
        nc = len(C)
    S = np.empty((r, nc))
    lib().ora_wtx_cols(_ptr(W), xf, xd, m, n, r, _ptr(C), nc, _ptr(S))
    return S


def h_update_cols(Hcols: np.ndarray, S: np.ndarray, G: np.ndarray, eps: float = 1e-16) -> np.ndarray:
    """H <- H*S / (G H + eps) on a column slice (MU, reading R1-R4)."""
    Hc = np.array(Hcols, dtype=np.float64, order="C", copy=True)
    r, nc = Hc.shape
    S = np.ascontiguousarray(S, dtype=np.float64)
    G = np.ascontiguousarray(G, dtype=np.float64)
    lib().ora_h_update_cols(_ptr(Hc), nc, r, _ptr(S), _ptr(G), eps)
    return Hc


def objective(X: np.ndarray, W: np.ndarray, H: np.ndarray) -> float:
    """1/2 ||X - WH||_F^2 by direct differences (Alg. 3 l.16)."""
    X, xf, xd = _xargs(X)
    m, n = X.shape
    W = np.ascontiguousarray(W, dtype=np.float64)
    H = np.ascontiguousarray(H, dtype=np.float64)
    return float(lib().ora_objective(xf, xd, m, n, W.shape[1], _ptr(W), _ptr(H)))


def nmf_mu(X: np.ndarray, W0: np.ndarray, H0: np.ndarray, iters: int, eps: float = 1e-16,
           trace: bool = False):
    """MU NMF from (W0, H0) for `iters` iterations (W half then H half).
    Returns (W, H) or (W, H, objective_trace)."""
    X, xf, xd = _xargs(X)
    m, n = X.shape
    W = np.array(W0, dtype=np.float64, order="C", copy=True)
    H = np.array(H0, dtype=np.float64, order="C", copy=True)
    r = W.shape[1]
    assert W.shape == (m, r) and H.shape == (r, n)
    tr = np.empty(iters) if trace else None
    _check(lib().ora_nmf_mu(xf, xd, m, n, r, iters, eps, _ptr(W), _ptr(H), _ptr(tr)))
    return (W, H, tr) if trace else (W, H)


# -------------------------------------------------------------- nTT sweep --
def check_ranks(dims, ranks) -> int:
    D, R = _dims(dims), _ranks(ranks)
    return int(lib().ora_check_ranks(len(D), _ptr(D), _ptr(R)))


def ntt_decompose(A: np.ndarray, ranks, iters: int, seed: int = 0, eps: float = 1e-16) -> np.ndarray:
    """Alg. 2 with fixed ranks and MU NMF; returns packed fp64 cores."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    D, R = _dims(A.shape), _ranks(ranks)
    cores = np.empty(cores_size(list(A.shape), list(ranks)))
    _check(lib().ora_ntt_decompose(_ptr(A), len(D), _ptr(D), _ptr(R), iters, seed, eps, _ptr(cores)))
    return cores


def unpack_cores(dims, ranks, cores: np.ndarray):
    """Split the packed buffer into the d cores, core l of shape (r_{l-1}, n_l, r_l)."""
    full = [1, *ranks, 1]
    out, off = [], 0
    for l in range(len(dims)):
        sz = full[l] * dims[l] * full[l + 1]
        out.append(np.asarray(cores[off:off + sz]).reshape(full[l], dims[l], full[l + 1]))
        off += sz
    return out


def rel_error(A: np.ndarray, B: np.ndarray) -> float:
    """Eq. 3 by direct differences."""
    Bd = np.ascontiguousarray(B, dtype=np.float64).ravel()
    if A.dtype == np.float32:
        Af = np.ascontiguousarray(A).ravel()
        return float(lib().ora_rel_error_f32(_ptr(Af), _ptr(Bd), Af.size))
    Ad = np.ascontiguousarray(A, dtype=np.float64).ravel()
    return float(lib().ora_rel_error(_ptr(Ad), _ptr(Bd), Ad.size))


def tt_rel_error(A: np.ndarray, ranks, cores: np.ndarray) -> float:
    """Eq. 3 of the TT reconstruction against fp32 A, element by element via Eq. 2's
    sequential vector-matrix products (no materialised reconstruction)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    D, R = _dims(A.shape), _ranks(ranks)
    C = np.ascontiguousarray(cores, dtype=np.float64)
    return float(lib().ora_tt_rel_error_f32(len(D), _ptr(D), _ptr(R), _ptr(C), _ptr(A)))


def tt_rel_error_split(A: np.ndarray, ranks, cores: np.ndarray, k: Optional[int] = None) -> float:
    """Eq. 3 with the reconstruction formed on the fly from Eq. 1 split at bond k
    (A~ = L_k R_k, fp64): the full-size evaluation (8 FMAs per element at r_k = 8)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    D, R = _dims(A.shape), _ranks(ranks)
    C = np.ascontiguousarray(cores, dtype=np.float64)
    kk = len(D) // 2 if k is None else k
    v = float(lib().ora_tt_rel_error_split_f32(len(D), _ptr(D), _ptr(R), _ptr(C), _ptr(A), kk))
    if v < -1.5:
        raise OracleError("tt_rel_error_split failed")
    return v


def compression_ratio(dims, ranks) -> float:
    """Eq. 4."""
    D, R = _dims(dims), _ranks(ranks)
    return float(lib().ora_compression_ratio(len(D), _ptr(D), _ptr(R)))


# ------------------------------------------- SVD rank rule (SURVEY s.8(f) f2) --
def svd_tail_rank(X: np.ndarray, tt_eps: float, rmax: Optional[int] = None) -> int:
    """Alg. 2 l.5-6 and section III-A: r = the smallest k in
    [1, N], N = min(m, n), with sqrt(s_{k+1}^2 + ... + s_N^2) / sqrt(s_1^2 + ... + s_N^2)
    <= eps.  Singular values by LAPACK (numpy.linalg.svd -- a library primitive used
    as one step, SURVEY s.8(c)); the tail sums are accumulated from the smallest
    value up.  Optional cap rmax (reading R21).  An all-zero X gives r = 1."""
    s = np.linalg.svd(np.asarray(X, dtype=np.float64), compute_uv=False)
    e = s * s
    N = e.size
    tot = float(e.sum())
    if tot == 0.0:
        return 1
    # tail[k] = sum_{i > k} e_i (1-based k), k = 1..N
    asc = np.cumsum(e[::-1])          # asc[j-1] = sum of the j smallest
    r = N
    for k in range(1, N + 1):
        tail = float(asc[N - k - 1]) if k < N else 0.0
        if np.sqrt(tail / tot) <= tt_eps:
            r = k
            break
    return min(r, rmax) if rmax else r


def ntt_decompose_eps(A: np.ndarray, tt_eps: float, iters: int, seed: int = 0, eps: float = 1e-16,
                      max_ranks: Optional[Sequence[int]] = None):
    """Alg. 2 with the SVD rank rule of l.5-6 at every step (ranks chosen
    from the current unfolding X_l = reshape(H_{l-1})) and MU NMF (R1-R4); inits as
    ntt_decompose (streams 0x200 + 2l / 0x201 + 2l).  Returns (ranks, packed fp64 cores)."""
    A = np.ascontiguousarray(A, dtype=np.float32)
    dims = list(A.shape)
    d = len(dims)
    T = A.reshape(-1)
    rprev = 1
    ranks, cores = [], []
    rest = T.size
    for l in range(1, d):
        m = rprev * dims[l - 1]
        rest //= dims[l - 1]
        n = rest
        X = T.reshape(m, n)
        cap = min(m, n, max_ranks[l - 1]) if max_ranks else min(m, n)
        r = svd_tail_rank(X, tt_eps, cap)
        W0 = fill_uniform(m * r, seed, stream_w(l)).reshape(m, r)
        H0 = fill_uniform(r * n, seed, stream_h(l)).reshape(r, n)
        W, H = nmf_mu(X, W0, H0, iters, eps)
        cores.append(W.reshape(-1))
        ranks.append(r)
        T = H.reshape(-1)
        rprev = r
    cores.append(T)
    return ranks, np.concatenate(cores)


# ------------------------------------------------- BCD NMF (SURVEY s.8(f) f1) --
def _spec(M: np.ndarray) -> float:
    """Spectral norm of a symmetric PSD r x r Gram (LAPACK eigvalsh, a library primitive)."""
    return float(np.linalg.eigvalsh(np.asarray(M, np.float64))[-1]) if M.size else 0.0


def nmf_bcd(X: np.ndarray, W0: np.ndarray, H0: np.ndarray, iters: int, delta: float = 0.9999,
            trace: bool = False, log: Optional[list] = None, force_correct=()):
    """Alg. 3 (distBCDnmf) on one process, fp64, with readings
    R22-R27 (DESIGN.md s.3):
      init  W_m = W0 sqrt(||X||_F)/||W0||_F, H_m = H0 sqrt(||X||_F)/||H0||_F; W = W_m, H = H_m;
            Q = H H^T, P = X H^T, t = 1, obj = 1/2 ||X||_F^2, L_W(prev) = ||Q||_2, L_H(prev) = ||W^T W||_2
      loop  W  = max(0, W_m - (W_m Q - P) / L_W),  L_W = ||Q||_2           (l.6-8)
            column L1 normalisation of W: c_k = sum_i W[i][k] (> 0): W[:, k] /= c_k,
            H_m[k, :] *= c_k, H_prev[k, :] *= c_k, W_prev[:, k] /= c_k     (l.9; WH invariant)
            G  = W^T W,  L_H = ||G||_2                                      (l.10)
            H  = max(0, H_m - (G H_m - W^T X) / L_H)                        (l.11-14)
            Q = H H^T, P = X H^T, obj_new = 1/2 ||X - W H||_F^2             (l.15-16)
            obj_new >= obj: correction -- back to the last accepted (W_prev, H_prev),
                W_m = W_prev, H_m = H_prev, t = 1, Q, P from H_prev         (l.17-20)
            else extrapolation: t+ = (1 + sqrt(1 + 4 t^2)) / 2, w = (t - 1) / t+,
                w_W = min(w, delta sqrt(L_W_prev / L_W)), w_H = min(w, delta sqrt(L_H_prev / L_H)),
                W_m = W + w_W (W - W_prev), H_m = H + w_H (H - H_prev),
                W_prev, H_prev = W, H; L_*_prev = L_*; t = t+; obj = obj_new  (l.21-27)
    Returns (W, H) = the last accepted iterates, or (W, H, accepted-objective trace).
    Test instrumentation (tests/test_oracle_bcd.py pins these against the hand-worked
    tests/golden/bcd_worked.json): ``log`` (a list) receives one dict per iteration with the
    scalars of the iteration (L_W, L_H, c, obj_new, the branch, t before / after, w, w_W, w_H);
    ``force_correct`` holds 0-based iteration indices whose l.17 test is treated as true
    (a constructed overshoot for the correction branch, l.17-20)."""
    X = np.asarray(X, dtype=np.float64)
    m, n = X.shape
    W0 = np.asarray(W0, dtype=np.float64)
    H0 = np.asarray(H0, dtype=np.float64)
    r = W0.shape[1]
    nx = np.linalg.norm(X)
    if nx == 0.0:
        raise ValueError("||X|| = 0 (DegenerateInputError, S:330)")
    if np.linalg.norm(W0) == 0.0 or np.linalg.norm(H0) == 0.0:
        raise ValueError("||W0|| = 0 or ||H0|| = 0: l.2 cannot normalise (DegenerateInputError, S:330)")
    Wm = W0 * (np.sqrt(nx) / np.linalg.norm(W0))
    Hm = H0 * (np.sqrt(nx) / np.linalg.norm(H0))
    Wp, Hp = Wm.copy(), Hm.copy()
    Q, P = Hp @ Hp.T, X @ Hp.T
    t, obj = 1.0, 0.5 * nx * nx
    LWp, LHp = _spec(Q), _spec(Wp.T @ Wp)
    tr = []
    for _ in range(iters):
        LW = _spec(Q)
        W = np.maximum(0.0, Wm - (Wm @ Q - P) / LW) if LW > 0 else Wm.copy()
        c = W.sum(axis=0)
        nz = c > 0
        W[:, nz] /= c[nz]
        Hm = Hm.copy()
        Hp = Hp.copy()
        Wp = Wp.copy()
        Hm[nz, :] *= c[nz, None]
        Hp[nz, :] *= c[nz, None]
        Wp[:, nz] /= c[nz]
        G = W.T @ W
        LH = _spec(G)
        H = np.maximum(0.0, Hm - (G @ Hm - W.T @ X) / LH) if LH > 0 else Hm.copy()
        obj_new = 0.5 * float(np.sum((X - W @ H) ** 2))
        ent = dict(it=len(tr), LW=LW, LH=LH, c=c.tolist(), obj_new=obj_new, t=t)
        if obj_new >= obj or len(tr) in force_correct:      # correction
            Wm, Hm, t = Wp.copy(), Hp.copy(), 1.0
            Q, P = Hp @ Hp.T, X @ Hp.T
            ent.update(accepted=False)
        else:                       # extrapolation
            tp = (1.0 + np.sqrt(1.0 + 4.0 * t * t)) / 2.0
            w = (t - 1.0) / tp
            wW = min(w, delta * np.sqrt(LWp / LW))
            wH = min(w, delta * np.sqrt(LHp / LH))
            Wm = W + wW * (W - Wp)
            Hm = H + wH * (H - Hp)
            Wp, Hp = W, H
            LWp, LHp = LW, LH
            t, obj = tp, obj_new
            Q, P = H @ H.T, X @ H.T
            ent.update(accepted=True, w=w, wW=wW, wH=wH)
        if log is not None:
            ent.update(t_next=t, W=Wp.copy(), H=Hp.copy(), Wm=Wm.copy(), Hm=Hm.copy())
            log.append(ent)
        tr.append(obj)
    return (Wp, Hp, np.array(tr)) if trace else (Wp, Hp)


# ---------------------------------------------- TT-SVD baseline (SURVEY s.8(f) f4) --
def tt_svd(A: np.ndarray, tt_eps: float, max_ranks: Optional[Sequence[int]] = None):
    """Unconstrained TT by sequential truncated SVDs (TT-SVD, the baseline the paper compares
    nTT against: P:78), reading R28 (DESIGN.md s.3): at step l the current
    matrix X_l (r_{l-1} n_l x prod_{i>l} n_i, as Alg. 2 l.4) is factored by LAPACK's SVD
    (numpy.linalg.svd, a library primitive), r_l is chosen by the same tail rule as the nTT
    sweep (svd_tail_rank, Alg. 2 l.5-6, capped by max_ranks), core l = U[:, :r_l] and
    X_{l+1} = reshape(diag(s[:r_l]) V^T[:r_l]); the last core is X_d.  Sign convention (the
    SVD fixes singular vectors only up to sign): the largest-magnitude entry of every kept
    column of U is positive (lowest index on ties), the matching row of V^T flips with it.
    Returns (ranks, packed fp64 cores, per-step discarded energies sum_{i > r_l} s_i^2)."""
    A = np.asarray(A, dtype=np.float64)
    dims = list(A.shape)
    d = len(dims)
    T = A.reshape(-1)
    rprev, rest = 1, T.size
    ranks, cores, tails = [], [], []
    for l in range(1, d):
        m = rprev * dims[l - 1]
        rest //= dims[l - 1]
        X = T.reshape(m, rest)
        cap = min(m, rest, max_ranks[l - 1]) if max_ranks else min(m, rest)
        r = svd_tail_rank(X, tt_eps, cap)
        U, s, Vt = np.linalg.svd(X, full_matrices=False)
        U, s, Vt = U[:, :r].copy(), s.copy(), Vt[:r].copy()
        for k in range(r):
            i = int(np.argmax(np.abs(U[:, k])))
            if U[i, k] < 0:
                U[:, k] = -U[:, k]
                Vt[k] = -Vt[k]
        tails.append(float(np.sum(s[r:] ** 2)))
        cores.append(U.reshape(-1))
        ranks.append(r)
        T = (s[:r, None] * Vt).reshape(-1)
        rprev = r
    cores.append(T)
    return ranks, np.concatenate(cores), np.array(tails)


def ntt_decompose_bcd(A: np.ndarray, ranks, iters: int, seed: int = 0, delta: float = 0.9999) -> np.ndarray:
    """Alg. 2 with fixed ranks and the paper's own NMF, BCD (Alg. 3 via nmf_bcd,
    readings R22-R27), at every step: inits W0, H0 from the streams of R20 (as ntt_decompose),
    core l = W_l, next X = reshape(H_l) (Alg. 2 l.8-10).  Returns packed fp64 cores."""
    A = np.asarray(A, dtype=np.float64)
    dims = list(A.shape)
    d = len(dims)
    T = A.reshape(-1)
    rprev, rest = 1, T.size
    cores = []
    for l in range(1, d):
        m = rprev * dims[l - 1]
        rest //= dims[l - 1]
        r = int(ranks[l - 1])
        X = T.reshape(m, rest)
        W0 = fill_uniform(m * r, seed, stream_w(l)).reshape(m, r)
        H0 = fill_uniform(r * rest, seed, stream_h(l)).reshape(r, rest)
        W, H = nmf_bcd(X, W0, H0, iters, delta)
        cores.append(W.reshape(-1))
        T = H.reshape(-1)
        rprev = r
    cores.append(T)
    return np.concatenate(cores)
