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


# ----------------------------------------------------------------------------------------
# Hand-worked iterations (tests/golden/bcd_worked.json): the scalars of every iteration --
# Lipschitz constants, l.9 scales, objective, branch, t, w, w_W, w_H -- and the iterates,
# including a correction (l.17-20) followed by extrapolations.
import json
import os

_GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "bcd_worked.json")


def _golden():
    with open(_GOLD) as f:
        return json.load(f)


def _close(a, b, rel=1e-13):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.all(np.abs(a - b) <= rel * np.maximum(1.0, np.abs(b)))


@pytest.mark.parametrize("name", ["A", "B", "C"])
def test_bcd_hand_worked(ora, name):
    g = _golden()
    case = next(c for c in g["cases"] if c["name"] == name)
    X = np.array(g["inputs"]["X"], np.float64)
    W0 = np.array([[3 / 5], [4 / 5]])
    H0 = np.array([[12 / 25, 3 / 5, 16 / 25]])
    log = []
    W, H = ora.nmf_bcd(X, W0, H0, case["iters"], delta=case["delta"], log=log,
                       force_correct=set(case["force_correct"]))
    assert len(log) == case["iters"]
    for e, ref in zip(log, case["iterations"]):
        it = ref["it"]
        assert e["accepted"] == ref["accepted"], it
        for k in ("LW", "LH", "obj_new", "t", "t_next"):
            assert _close(e[k], ref[k]), (it, k, e[k], ref[k])
        assert _close(e["c"], [ref["c"]]), (it, "c")
        if ref["accepted"]:
            for k in ("w", "wW", "wH"):
                assert _close(e[k], ref[k]), (it, k, e[k], ref[k])
        for k in ("W_prev", "H_prev", "Wm", "Hm"):
            ours = {"W_prev": e["W"], "H_prev": e["H"], "Wm": e["Wm"], "Hm": e["Hm"]}[k]
            assert _close(np.ravel(ours), ref[k]), (it, k)
    last = case["iterations"][-1]
    assert _close(W.ravel(), last["W_prev"]) and _close(H.ravel(), last["H_prev"])


def test_bcd_t_sequence(ora):
    """Case A: t_1 = 1, t_{k+1} = (1 + sqrt(1 + 4 t_k^2)) / 2, so
    t_2 = golden ratio, t_3 = 2.1935270853310539; w_k = (t_k - 1) / t_{k+1} (l.22, not
    (t_k - 1) / t_k)."""
    g = _golden()
    it = next(c for c in g["cases"] if c["name"] == "A")["iterations"]
    assert abs(it[0]["t_next"] - (1 + 5 ** 0.5) / 2) < 1e-15
    assert abs(it[1]["t_next"] - 2.1935270853310539) < 1e-15
    assert abs(it[1]["w"] - 0.2817535251253208) < 1e-15
    assert abs(it[1]["w"] - ((1 + 5 ** 0.5) / 2 - 1) / ((1 + 5 ** 0.5) / 2)) > 0.1


def test_bcd_correction_returns_to_last_accepted(ora):
    """l.17-20 (reading R26): a correction discards (W, H) of the iteration, sets
    W_m = W_prev, H_m = H_prev (the last accepted iterate, after the l.9 rescale), t = 1
    and recomputes P, Q from H_prev; the accepted objective does not move.  With r = 3 the
    next iteration's prox steps depend on W_m and H_m, so they must equal those of a run
    whose extrapolation weights are zero at that point (w = (1 - 1)/t_+ = 0)."""
    rng = np.random.default_rng(11)
    X = rng.random((9, 14))
    W0, H0 = inits(9, 14, 3, 11)
    log = []
    _, _, tr = ora.nmf_bcd(X, W0, H0, 6, log=log, force_correct={3}, trace=True)
    e3, e2 = log[3], log[2]
    assert not e3["accepted"] and e3["t_next"] == 1.0
    c = np.asarray(e3["c"])
    # W_m / H_m after the correction = the accepted iterate of iteration 2, rescaled by c (l.9)
    assert np.allclose(e3["Wm"], e2["W"] / c, rtol=1e-14, atol=0)
    assert np.allclose(e3["Hm"], e2["H"] * c[:, None], rtol=1e-14, atol=0)
    assert np.array_equal(e3["W"], e3["Wm"]) and np.array_equal(e3["H"], e3["Hm"])
    assert tr[3] == tr[2]
    # iteration 4 starts with t = 1: w = 0, so W_m of iteration 4 is its own W
    assert log[4]["accepted"] and log[4]["w"] == 0.0 and log[4]["wW"] == 0.0
    assert np.array_equal(log[4]["Wm"], log[4]["W"])


def test_bcd_natural_corrections_occur(ora):
    """The correction branch is not only a hook: on the GPU parity inputs of
    tests/test_gpu_bcd.py::test_bcd_correction_parity the l.17 test fires by itself; the
    accepted objective never increases across them."""
    for m, n, r, seed, kind, iters in [(7, 64, 3, 11, "scaled", 52), (7, 64, 3, 10, "colscaled", 63)]:
        X = ni.bcd_overshoot_matrix(m, n, r, seed, kind).astype(np.float64)
        W0, H0 = inits(m, n, r, seed)
        log = []
        _, _, tr = ora.nmf_bcd(X, W0, H0, iters, log=log, trace=True)
        corr = [e for e in log if not e["accepted"]]
        assert len(corr) >= 2
        assert all(e["obj_new"] >= tr[e["it"]] for e in corr)     # a real overshoot
        assert all(log[e["it"] + 1]["w"] == 0.0 for e in corr if e["it"] + 1 < iters)
    assert np.all(np.diff(tr) <= 0.0)
