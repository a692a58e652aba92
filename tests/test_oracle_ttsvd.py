"""Pins of the oracle's TT-SVD baseline (SURVEY s.8(f) f4; reading R28):
facts the mathematics fixes independently of the implementation.

* Eckart-Young: for d = 2 TT-SVD is the truncated SVD, so the error equals the
  discarded singular-value energy and no rank-r matrix does better (checked against
  random rank-r competitors).
* Orthogonality: every core but the last, reshaped to (r_{l-1} n_l) x r_l, has orthonormal
  columns, and the squared error is exactly the sum of the per-step discarded energies.
* Exact recovery: a tensor of TT ranks (r_1..r_{d-1}) is reproduced to rounding when the
  caps allow those ranks (eps = 0), and the chosen ranks equal the true ones for small eps.
* The sign convention: the largest-magnitude entry of every core column is positive."""
import numpy as np
import pytest


def rand_tt(dims, ranks, seed):
    rng = np.random.default_rng(seed)
    rr = [1] + list(ranks) + [1]
    out = None
    for l, n in enumerate(dims):
        G = rng.standard_normal((rr[l], n, rr[l + 1]))
        out = G.reshape(n, -1) if out is None else (out.reshape(-1, rr[l]) @ G.reshape(rr[l], -1))
    return out.reshape(dims)


def test_d2_is_truncated_svd(ora):
    rng = np.random.default_rng(0)
    A = rng.standard_normal((30, 50))
    s = np.linalg.svd(A, compute_uv=False)
    for eps in (0.9, 0.5, 0.2):
        ranks, cores, tails = ora.tt_svd(A, eps)
        B = ora.tt_full(list(A.shape), ranks, cores)
        err2 = float(np.sum((A - B) ** 2))
        r = ranks[0]
        assert abs(err2 - float(np.sum(s[r:] ** 2))) <= 1e-10 * float(np.sum(s ** 2))
        assert np.sqrt(float(np.sum(s[r:] ** 2)) / float(np.sum(s ** 2))) <= eps
        for t in range(5):  # no rank-r competitor beats it
            C = rng.standard_normal((30, r)) @ rng.standard_normal((r, 50))
            Cb = C * (np.sum(A * C) / np.sum(C * C))
            assert float(np.sum((A - Cb) ** 2)) >= err2


@pytest.mark.parametrize("dims,eps", [((6, 5, 7, 4), 0.3), ((4, 4, 4, 4, 4), 0.2), ((3, 8, 5), 0.05)])
def test_orthonormal_cores_and_error_decomposition(ora, dims, eps):
    rng = np.random.default_rng(sum(dims))
    A = rng.random(dims)
    ranks, cores, tails = ora.tt_svd(A, eps)
    parts = ora.unpack_cores(list(dims), ranks, cores)
    for l, G in enumerate(parts[:-1]):
        M = G.reshape(-1, G.shape[-1])
        assert np.allclose(M.T @ M, np.eye(M.shape[1]), atol=1e-12)
        j = np.argmax(np.abs(M), axis=0)
        assert np.all(M[j, np.arange(M.shape[1])] > 0)
    B = ora.tt_full(list(dims), ranks, cores)
    err2 = float(np.sum((A - B) ** 2))
    assert abs(err2 - tails.sum()) <= 1e-10 * float(np.sum(A ** 2))
    # each step meets the rule on its own matrix, so the error is <= eps * sqrt(d - 1) ||A||
    assert np.sqrt(err2) <= eps * np.sqrt(len(dims) - 1) * np.linalg.norm(A) * (1 + 1e-12)


@pytest.mark.parametrize("dims,tr", [((5, 6, 4, 7), (2, 3, 2)), ((4, 4, 4, 4, 4), (3, 4, 4, 2))])
def test_exact_tt_recovery(ora, dims, tr):
    A = rand_tt(dims, tr, 7)
    ranks, cores, tails = ora.tt_svd(A, 1e-9)
    assert list(ranks) == list(tr)
    B = ora.tt_full(list(dims), ranks, cores)
    assert np.abs(A - B).max() <= 1e-10 * np.abs(A).max()
    ranks0, cores0, _ = ora.tt_svd(A, 0.0, max_ranks=[64] * (len(dims) - 1))   # full ranks
    assert np.abs(A - ora.tt_full(list(dims), ranks0, cores0)).max() <= 1e-10 * np.abs(A).max()


def test_caps_and_rank_one(ora):
    a, b, c = np.arange(1, 7.0), np.array([2.0, -1.0]), np.arange(1, 5.0)
    A = np.einsum("i,j,k->ijk", a, b, c)
    ranks, cores, tails = ora.tt_svd(A, 1e-12)
    assert ranks == [1, 1]
    assert np.allclose(ora.tt_full([6, 2, 4], ranks, cores), A, rtol=0, atol=1e-12)
    G1 = cores[:6]
    assert np.allclose(G1, a / np.linalg.norm(a))          # positive-max sign convention
    rng = np.random.default_rng(1)
    B = rng.random((6, 5, 4))
    ranks, cores, _ = ora.tt_svd(B, 0.0, max_ranks=[2, 3])
    assert ranks == [2, 3]
    ranks, cores, _ = ora.tt_svd(B, 0.0)
    assert ranks == [6, 4]                                  # min(m, n) at every step
