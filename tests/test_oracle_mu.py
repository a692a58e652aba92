"""Oracle pins: the MU NMF iteration (readings R1-R4, R18).

Each test pins the oracle to something outside itself: a hand-worked example
(golden), the Eckart-Young theorem via numpy's SVD, the rank-1 closed form, the
Lee-Seung monotonicity theorem, exact fixed points, exact power-of-two scale
invariance, the transpose duality between the W and H half-steps, numpy matmul
for the products, and exact rational arithmetic on tiny integer inputs.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "mu_worked_2x2.json")))


def _fr(s):
    return float(Fraction(s))


def test_worked_2x2_example(ora):
    X = np.array(GOLD["X"], float)
    W, H, tr = ora.nmf_mu(X, np.array(GOLD["W0"], float), np.array(GOLD["H0"], float), 1, eps=GOLD["eps"],
                          trace=True)
    assert W.ravel().tolist() == pytest.approx([_fr(s[0]) for s in GOLD["W1"]], rel=1e-15)
    assert H.ravel().tolist() == pytest.approx([_fr(s) for s in GOLD["H1"][0]], rel=1e-15)
    assert ora.objective(X, np.array(GOLD["W0"], float), np.array(GOLD["H0"], float)) == float(GOLD["obj0"])
    assert tr[0] == pytest.approx(_fr(GOLD["obj1"]), rel=1e-14)


def test_worked_2x2_converges_to_eckart_young(ora):
    X = np.array(GOLD["X"], float)
    W, H, tr = ora.nmf_mu(X, np.array(GOLD["W0"], float), np.array(GOLD["H0"], float), 60, eps=0.0, trace=True)
    limit = 0.5 * (15 - math.sqrt(221))
    assert tr[-1] == pytest.approx(limit, rel=1e-12)
    s = np.linalg.svd(X, compute_uv=False)
    assert limit == pytest.approx(0.5 * s[1] ** 2, rel=1e-12)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_r1_limit_is_eckart_young(ora, seed):
    rng = np.random.default_rng(seed)
    X = rng.random((7, 9)) + 0.1  # positive: Perron vectors, MU r=1 -> best rank-1
    W, H, tr = ora.nmf_mu(X, rng.random((7, 1)) + 0.1, rng.random((1, 9)) + 0.1, 400, eps=0.0, trace=True)
    s = np.linalg.svd(X, compute_uv=False)
    assert tr[-1] == pytest.approx(0.5 * (s[1:] ** 2).sum(), rel=1e-9)


def test_rank1_one_step_closed_form(ora):
    rng = np.random.default_rng(4)
    a, v = rng.random(11) + 0.05, rng.random(13) + 0.05
    X = np.outer(a, v)
    W, H = ora.nmf_mu(X, rng.random((11, 1)) + 0.05, rng.random((1, 13)) + 0.05, 1, eps=0.0)
    assert np.allclose(W @ H, X, rtol=1e-13, atol=0)
    # W1 is proportional to a
    ratio = W[:, 0] / a
    assert np.allclose(ratio, ratio[0], rtol=1e-13)


@pytest.mark.parametrize("m,n,r,seed", [(20, 30, 3, 0), (8, 50, 5, 1), (40, 12, 4, 2)])
def test_monotone_and_nonnegative(ora, m, n, r, seed):
    rng = np.random.default_rng(seed)
    X = rng.random((m, n))
    W0, H0 = rng.random((m, r)), rng.random((r, n))
    obj0 = ora.objective(X, W0, H0)
    W, H, tr = ora.nmf_mu(X, W0, H0, 150, eps=0.0, trace=True)
    seq = np.concatenate([[obj0], tr])
    assert np.all(np.diff(seq) <= 1e-12 * seq[:-1])  # Lee-Seung: non-increasing
    assert seq[-1] < 0.5 * seq[0]
    assert np.all(W >= 0) and np.all(H >= 0)


def test_fixed_point(ora):
    rng = np.random.default_rng(5)
    Ws, Hs = rng.random((9, 2)) + 0.1, rng.random((2, 14)) + 0.1
    X = Ws @ Hs
    W, H = ora.nmf_mu(X, Ws, Hs, 5, eps=0.0)
    assert np.allclose(W, Ws, rtol=1e-13) and np.allclose(H, Hs, rtol=1e-13)


def test_scale_invariance_bit_exact(ora):
    rng = np.random.default_rng(6)
    X = rng.random((12, 17))
    W0, H0 = rng.random((12, 3)), rng.random((3, 17))
    W, H = ora.nmf_mu(X, W0, H0, 7, eps=0.0)
    W8, H8 = ora.nmf_mu(8.0 * X, W0, H0, 7, eps=0.0)
    # P, S scale by 8 and 64, denominators by 1 and 64: powers of two are exact
    assert np.array_equal(W8, 8.0 * W)
    assert np.array_equal(H8, H)


def test_building_blocks_vs_numpy(ora):
    rng = np.random.default_rng(7)
    X = rng.random((13, 29))
    W, H = rng.random((13, 4)), rng.random((4, 29))
    assert np.allclose(ora.xht(X, H), X @ H.T, rtol=1e-14)
    assert np.allclose(ora.gram_rows(H), H @ H.T, rtol=1e-14)
    assert np.allclose(ora.gram_cols(W), W.T @ W, rtol=1e-14)
    assert np.allclose(ora.wtx_cols(W, X), W.T @ X, rtol=1e-14)
    cols = [3, 0, 28, 11]
    assert np.allclose(ora.wtx_cols(W, X, cols), (W.T @ X)[:, cols], rtol=1e-14)
    Xf = X.astype(np.float32)
    assert np.allclose(ora.xht(Xf, H), Xf.astype(np.float64) @ H.T, rtol=1e-14)
    P, Q = X @ H.T, H @ H.T
    assert np.allclose(ora.w_update(W, P, Q, 0.0), W * P / (W @ Q), rtol=1e-14)
    G, S = W.T @ W, W.T @ X
    assert np.allclose(ora.h_update_cols(H, S, G, 0.0), H * S / (G @ H), rtol=1e-14)


def test_transpose_duality_bit_exact(ora):
    """The H half-step on X equals the W half-step on X^T with roles swapped."""
    rng = np.random.default_rng(8)
    X = rng.random((10, 15))
    W, H = rng.random((10, 3)), rng.random((3, 15))
    G = ora.gram_cols(W)
    S = ora.wtx_cols(W, X)
    Hn = ora.h_update_cols(H, S, G, 1e-16)
    Wt = ora.w_update(H.T, ora.xht(X.T, W.T), G, 1e-16)
    assert np.array_equal(Wt.T, Hn)
    assert np.array_equal(ora.xht(X, H), ora.wtx_cols(H.T, X.T).T)


def test_zero_row_stays_zero_with_eps(ora):
    """eps only guards 0/0 (reading R3): a zero W row stays exactly zero."""
    rng = np.random.default_rng(9)
    X = rng.random((6, 8))
    W0, H0 = rng.random((6, 2)), rng.random((2, 8))
    W0[2, :] = 0.0
    X[2, :] = 0.0
    W, H = ora.nmf_mu(X, W0, H0, 5, eps=1e-16)
    assert np.all(W[2] == 0) and np.all(np.isfinite(W)) and np.all(np.isfinite(H))


def _mu_exact(X, W, H, iters):
    m, n = len(X), len(X[0])
    r = len(W[0])
    for _ in range(iters):
        P = [[sum(X[i][j] * H[k][j] for j in range(n)) for k in range(r)] for i in range(m)]
        Q = [[sum(H[k][j] * H[l][j] for j in range(n)) for l in range(r)] for k in range(r)]
        D = [[sum(W[i][l] * Q[l][k] for l in range(r)) for k in range(r)] for i in range(m)]
        W = [[W[i][k] * P[i][k] / D[i][k] for k in range(r)] for i in range(m)]
        G = [[sum(W[i][k] * W[i][l] for i in range(m)) for l in range(r)] for k in range(r)]
        S = [[sum(W[i][k] * X[i][j] for i in range(m)) for j in range(n)] for k in range(r)]
        E = [[sum(G[k][l] * H[l][j] for l in range(r)) for j in range(n)] for k in range(r)]
        H = [[H[k][j] * S[k][j] / E[k][j] for j in range(n)] for k in range(r)]
    return W, H


@pytest.mark.parametrize("seed", [0, 1])
def test_exact_rational_tiny(ora, seed):
    rng = np.random.default_rng(seed)
    Xi = rng.integers(1, 6, size=(2, 3))
    Wi = rng.integers(1, 4, size=(2, 2))
    Hi = rng.integers(1, 4, size=(2, 3))
    F = lambda A: [[Fraction(int(v)) for v in row] for row in A]
    We, He = _mu_exact(F(Xi), F(Wi), F(Hi), 3)
    W, H = ora.nmf_mu(Xi.astype(float), Wi.astype(float), Hi.astype(float), 3, eps=0.0)
    assert np.allclose(W, np.array(We, dtype=float), rtol=1e-14, atol=0)
    assert np.allclose(H, np.array(He, dtype=float), rtol=1e-14, atol=0)
