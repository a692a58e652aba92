"""Pins of the oracle's SVD tail-energy rank rule (Alg. 2 l.5-6, section
III-A P:194; SURVEY s.8(f) f2) and of the eps-driven sweep built on it."""
import numpy as np
import pytest

import ntt_inputs as ni


def spectrum_matrix(s, m=6, n=9, seed=0):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, len(s))))
    V, _ = np.linalg.qr(rng.standard_normal((n, len(s))))
    return (U * np.asarray(s, float)) @ V.T


# spectrum 10, 5, 1, 0.1, 0.01, 0.001: total energy 126.010101; the tail ratios after
# k = 1..5 are sqrt(26.010101/T) = 0.4543, sqrt(1.010101/T) = 0.08953,
# sqrt(0.010101/T) = 8.953e-3, sqrt(1.01e-4/T) = 8.953e-4, sqrt(1e-6/T) = 8.908e-5
@pytest.mark.parametrize("eps,r", [(2.0, 1), (0.5, 1), (0.45, 2), (0.2, 2), (0.09, 2), (0.0895, 3), (0.01, 3),
                                   (9e-4, 4), (8.95e-4, 5), (1e-4, 5), (8.9e-5, 6), (1e-5, 6), (0.0, 6)])
def test_rank_rule_on_known_spectrum(ora, eps, r):
    X = spectrum_matrix([10, 5, 1, 0.1, 0.01, 0.001])
    assert ora.svd_tail_rank(X, eps) == r
    assert ora.svd_tail_rank(X.T, eps) == r          # rule depends on the singular values only


def test_rank_rule_properties(ora):
    rng = np.random.default_rng(1)
    X = rng.random((12, 40))
    prev = None
    for eps in [1.0, 0.5, 0.2, 0.1, 0.05, 0.01, 1e-3, 1e-6, 0.0]:
        r = ora.svd_tail_rank(X, eps)
        assert 1 <= r <= 12
        if prev is not None:
            assert r >= prev                          # non-increasing in eps
        prev = r
    assert ora.svd_tail_rank(X, 0.0) == 12
    assert ora.svd_tail_rank(X, 1e-6, rmax=4) == 4
    assert ora.svd_tail_rank(np.zeros((3, 5)), 0.1) == 1


@pytest.mark.parametrize("k", [1, 2, 5])
def test_rank_rule_recovers_exact_rank(ora, k):
    rng = np.random.default_rng(k)
    X = rng.random((10, k)) @ rng.random((k, 30))    # non-negative, rank k exactly
    assert ora.svd_tail_rank(X, 1e-6) == k


def test_eps_sweep_matches_fixed_rank_sweep(ora):
    """The eps-driven sweep with the ranks it chose == the fixed-rank sweep (Alg. 2)."""
    dims, ranks = [5, 4, 5, 6], [4, 3, 2]
    A = ora.tt_full_f32(dims, ranks, ni.make_cores(dims, ranks, 0), noise_amp=0.05, seed=0)
    for eps in (0.3, 0.05, 0.01):
        got_r, got = ora.ntt_decompose_eps(A, eps, iters=5, seed=2)
        ref = ora.ntt_decompose(A, got_r, iters=5, seed=2)
        assert np.array_equal(got, ref)
        assert all(1 <= r for r in got_r)


def test_eps_sweep_first_rank_is_unfolding_rank(ora):
    """Step 1 sees X_1 = A unfolded; an exact rank-3 non-negative matrix (d = 2) gets r = 3."""
    rng = np.random.default_rng(4)
    A = (rng.random((7, 3)) @ rng.random((3, 11))).astype(np.float32)
    r, _ = ora.ntt_decompose_eps(A, 1e-5, iters=3)
    assert r == [3]
