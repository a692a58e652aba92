"""Oracle pins: the nTT sweep (Alg. 2 with fixed ranks).

Pinned by: the rank-1 TT closed form (exact after one MU iteration per step),
the d=2 reduction to a single NMF, a disjoint-support TT that MU
recovers exactly, core bookkeeping, rank validation, determinism across
thread counts.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import ntt_inputs as ni


def test_rank1_tt_exact_after_one_iteration(ora):
    dims = [5, 4, 6, 3, 2]
    # dyadic cores (k/8, k = 1..8) so the rank-1 tensor is exact in fp32
    cores = (np.floor(ni.make_cores(dims, [1] * 4, seed=3) * 8) + 1) / 8
    A = ora.tt_full_f32(dims, [1] * 4, cores)
    assert np.array_equal(A.astype(np.float64), ora.tt_full(dims, [1] * 4, cores))
    out = ora.ntt_decompose(A, [1] * 4, iters=1)
    assert ora.tt_rel_error(A, [1] * 4, out) < 1e-12
    assert np.all(out >= 0)


def test_d2_is_single_nmf(ora):
    dims, r = [7, 11], 3
    A = ora.tt_full_f32(dims, [r], ni.make_cores(dims, [r], seed=1), noise_amp=0.1, seed=1)
    cores = ora.ntt_decompose(A, [r], iters=25, seed=4)
    W0 = ni.uniform(7 * r, 4, ni.stream_w(1)).reshape(7, r)
    H0 = ni.uniform(r * 11, 4, ni.stream_h(1)).reshape(r, 11)
    W, H = ora.nmf_mu(A, W0, H0, 25)
    assert np.array_equal(cores[:7 * r], W.ravel())
    assert np.array_equal(cores[7 * r:], H.ravel())


def test_second_step_unfolds_first_H(ora):
    """Step 2's X is H_1 reshaped row-major to (r1 n2) x rest (Alg. 2 l.4/l.9)."""
    dims, ranks = [4, 3, 5], [2, 3]
    A = ora.tt_full_f32(dims, ranks, ni.make_cores(dims, ranks, seed=2))
    it = 6
    cores = ora.ntt_decompose(A, ranks, iters=it, seed=0)
    W0 = ni.uniform(4 * 2, 0, ni.stream_w(1)).reshape(4, 2)
    H0 = ni.uniform(2 * 15, 0, ni.stream_h(1)).reshape(2, 15)
    W1, H1 = ora.nmf_mu(A.reshape(4, 15), W0, H0, it)
    X2 = H1.reshape(2 * 3, 5)
    W0b = ni.uniform(6 * 3, 0, ni.stream_w(2)).reshape(6, 3)
    H0b = ni.uniform(3 * 5, 0, ni.stream_h(2)).reshape(3, 5)
    W2, H2 = ora.nmf_mu(X2, W0b, H0b, it)
    expect = np.concatenate([W1.ravel(), W2.ravel(), H2.ravel()])
    assert np.array_equal(cores, expect)


def test_disjoint_support_tt_recovered(ora):
    """G_l[k,i,k'] = delta_{kk'} g_l[k,i] with g_l[k,.] supported on block k of mode l:
    an exact, essentially-unique nonnegative factorisation; MU recovers it."""
    dims, r = [6, 6, 6, 6], 2
    rng = np.random.default_rng(11)
    parts = []
    fr = [1, r, r, r, 1]
    for l in range(4):
        G = np.zeros((fr[l], 6, fr[l + 1]))
        for k in range(r):
            blk = slice(3 * k, 3 * k + 3)
            if l == 0:
                G[0, blk, k] = rng.random(3) + 0.5
            elif l == 3:
                G[k, blk, 0] = rng.random(3) + 0.5
            else:
                G[k, blk, k] = rng.random(3) + 0.5
        parts.append(G.ravel())
    cores = np.concatenate(parts)
    A = ora.tt_full_f32(dims, [r] * 3, cores)
    out = ora.ntt_decompose(A, [r] * 3, iters=200, seed=0)
    assert ora.tt_rel_error(A, [r] * 3, out) < 1e-6


def test_config1_error_and_nonnegativity(ora):
    w = ni.workloads()["config1"]
    A = ora.tt_full_f32(w.dims, w.ranks, ni.make_cores(w.dims, w.ranks, w.seed))
    cores = ora.ntt_decompose(A, w.ranks, iters=w.iters, seed=w.seed)
    assert np.all(cores >= 0) and np.all(np.isfinite(cores))
    e = ora.tt_rel_error(A, w.ranks, cores)
    # MU "suffers from the inability to converge to a high accuracy":
    # the survey's probes land at 0.074-0.103 for this shape; our seed must too.
    assert 0.0 < e < 0.2
    assert ora.compression_ratio(w.dims, w.ranks) == pytest.approx(600 / 110)


def test_rank_validation(ora):
    assert ora.check_ranks([5, 4, 5, 6], [4, 3, 2]) == 0
    assert ora.check_ranks([5, 4, 5, 6], [6, 3, 2]) == 2     # r1 > n1
    assert ora.check_ranks([5, 4, 5, 6], [4, 17, 2]) == 2    # r2 > r1 n2 = 16
    assert ora.check_ranks([5, 4, 5, 6], [4, 3, 7]) == 2     # r3 > n4 = 6
    assert ora.check_ranks([5, 4, 5, 6], [4, 0, 2]) == 2
    assert ora.check_ranks([5], []) == 1                     # d < 2
    with pytest.raises(ora.OracleError):
        ora.ntt_decompose(np.ones((5, 4, 5, 6), np.float32), [6, 3, 2], 1)


def test_thread_count_invariance(ora, tmp_path):
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, oracle, ntt_inputs as ni\n"
        "w = ni.workloads()['config1']\n"
        "A = oracle.tt_full_f32(w.dims, w.ranks, ni.make_cores(w.dims, w.ranks, 0))\n"
        "c = oracle.ntt_decompose(A, w.ranks, 20)\n"
        "X = np.ascontiguousarray(A.reshape(20, 30).astype(np.float64))\n"
        "p = oracle.xht(X, np.ones((3, 30)))\n"
        "np.save(sys.argv[1], np.concatenate([c, p.ravel(), [oracle.tt_rel_error(A, w.ranks, c)]]))\n"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for th in ("1", "4"):
        f = str(tmp_path / f"o{th}.npy")
        env = dict(os.environ, OMP_NUM_THREADS=th)
        subprocess.check_call([sys.executable, "-c", code, f], env=env)
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])
