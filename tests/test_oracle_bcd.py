"""Pins of the oracle's BCD NMF (Alg. 3; readings R22-R27 in DESIGN.md;
SURVEY s.8(f) f1): properties the algorithm and the mathematics fix, and the paper's
claim that BCD reaches lower error than MU."""
import numpy as np
import pytest

import ntt_inputs as ni


def lowrank(m, n, r, seed):
    rng = np.random.default_rng(seed)
    return rng.random((m, r)) @ rng.random((r, n))


def inits(m, n, r, seed):
    return (ni.uniform(m * r, seed, ni.stream_w(1)).reshape(m, r),
            ni.uniform(r * n, seed, ni.stream_h(1)).reshape(r, n))


def relerr(X, W, H):
    return np.linalg.norm(X - W @ H) / np.linalg.norm(X)


def test_accepted_objective_nonincreasing_and_nonnegative(ora):
    rng = np.random.default_rng(3)
    X = rng.random((25, 60))
    W0, H0 = inits(25, 60, 4, 3)
    W, H, tr = ora.nmf_bcd(X, W0, H0, 200, trace=True)
    assert np.all(np.diff(tr) <= 0.0)
    assert tr[0] < 0.5 * np.linalg.norm(X) ** 2          # the first step descends from obj_0 = 1/2 ||X||^2
    assert np.all(W >= 0) and np.all(H >= 0)
    assert abs(tr[-1] - 0.5 * np.linalg.norm(X - W @ H) ** 2) <= 1e-12 * tr[-1]   # trace = accepted objective


def test_exact_rank_recovery(ora):
    """X = W* H* non-negative of rank 3: relative error <= 1e-4 within 500 iterations for >= 4 of 5 seeds."""
    ok = 0
    for seed in range(5):
        X = lowrank(30, 40, 3, seed)
        W0, H0 = inits(30, 40, 3, seed)
        W, H = ora.nmf_bcd(X, W0, H0, 500)
        ok += relerr(X, W, H) <= 1e-4
    assert ok >= 4


def test_bcd_beats_mu(ora):
    """BCD reaches a lower reconstruction error than MU (100 iterations, >= 4 of 5 seeds)."""
    wins = 0
    for seed in range(5):
        X = lowrank(20, 50, 4, 10 + seed) + 0.01 * np.random.default_rng(seed).random((20, 50))
        W0, H0 = inits(20, 50, 4, seed)
        Wb, Hb = ora.nmf_bcd(X, W0, H0, 100)
        Wm, Hm = ora.nmf_mu(X, W0, H0, 100)
        wins += relerr(X, Wb, Hb) <= relerr(X, Wm, Hm)
    assert wins >= 4


def test_rank1_fixed_point(ora):
    """X = u v^T started at (u, v^T): the normalised init reproduces X exactly (||u v^T||_F =
    ||u|| ||v||), the projected gradient is zero, and the iteration stays on X."""
    rng = np.random.default_rng(7)
    u, v = rng.random((9, 1)) + 0.1, rng.random((1, 13)) + 0.1
    X = u @ v
    W, H = ora.nmf_bcd(X, u, v, 20)
    assert np.linalg.norm(X - W @ H) <= 1e-12 * np.linalg.norm(X)
    assert np.allclose(W.sum(axis=0), 1.0)                 # L1-normalised columns (R24)


def test_rank1_random_init_converges(ora):
    rng = np.random.default_rng(8)
    X = (rng.random((12, 1)) + 0.1) @ (rng.random((1, 30)) + 0.1)
    W0, H0 = inits(12, 30, 1, 8)
    W, H = ora.nmf_bcd(X, W0, H0, 100)
    assert relerr(X, W, H) <= 1e-6


def test_column_normalisation_keeps_product(ora):
    """The L1 column normalisation with compensation (R24) leaves W H unchanged: the
    W columns of every accepted iterate have unit L1 norm."""
    rng = np.random.default_rng(9)
    X = rng.random((15, 35))
    W0, H0 = inits(15, 35, 3, 9)
    W, H = ora.nmf_bcd(X, W0, H0, 7)
    s = W.sum(axis=0)
    assert np.allclose(s[s > 0], 1.0)


def test_degenerate_input(ora):
    with pytest.raises(ValueError):
        ora.nmf_bcd(np.zeros((3, 4)), np.ones((3, 1)), np.ones((1, 4)), 2)


def test_ntt_bcd_sweep_pins(ora):
    """nTT with BCD at every step (Alg. 2 + Alg. 3): an exact rank-1 non-negative TT is
    recovered to rounding; on a non-negative TT with noise the BCD sweep reaches a lower
    error than the MU sweep at the same ranks and iterations (the paper's claim);
    factors stay non-negative."""
    rng = np.random.default_rng(4)
    vs = [rng.random(n) + 0.1 for n in (5, 4, 6, 3)]
    A1 = np.einsum("i,j,k,l->ijkl", *vs)
    c1 = ora.ntt_decompose_bcd(A1, [1, 1, 1], 50)
    assert ora.rel_error(A1, ora.tt_full([5, 4, 6, 3], [1, 1, 1], c1)) <= 1e-9
    dims, ranks = [6, 5, 7, 4], [3, 4, 2]
    A = ora.tt_full(dims, ranks, rng.random(ora.cores_size(dims, ranks))) + 0.05 * rng.random(dims)
    cb = ora.ntt_decompose_bcd(A, ranks, 100)
    cm = ora.ntt_decompose(A.astype(np.float32), ranks, 100)
    eb = ora.rel_error(A, ora.tt_full(dims, ranks, cb))
    em = ora.rel_error(A, ora.tt_full(dims, ranks, cm))
    assert np.all(cb >= 0) and eb < em
