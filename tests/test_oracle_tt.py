"""Oracle pins: TT contraction (Eq. 1 / Eq. 2), unfolding, Eq. 3, Eq. 4.

Pinned against SPEC.md's worked examples (tests/golden/spec_examples.json),
numpy einsum (a library routine as the independent reference), and the
literal Eq. 2 sum over k-tuples on tiny trains.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import ntt_inputs as ni

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_unfold_example_S56():
    g = GOLD["unfold_2x2x2"]
    t = np.array(g["data"]).reshape(g["shape"])
    X = t.reshape(g["rows"], -1)  # row-major unfolding (reading R8)
    assert X.tolist() == g["expect"]
    # 5x4x5x6, rows=5 -> row i is the contiguous slice starting at 120 i
    t = np.arange(600).reshape(5, 4, 5, 6)
    X = t.reshape(5, 120)
    for i in range(5):
        assert np.array_equal(X[i], np.arange(120 * i, 120 * i + 120))
    # round trip bit exact
    assert np.array_equal(X.reshape(5, 4, 5, 6), t)


def test_tt_element_examples(ora):
    g = GOLD["tt_element_ones"]
    dims, ranks = g["dims"], g["ranks"]
    cores = np.ones(ora.cores_size(dims, ranks))
    assert ora.tt_element(dims, ranks, cores, [2, 1, 3]) == g["expect"]
    g = GOLD["tt_element_outer"]
    assert ora.tt_element(g["dims"], g["ranks"], np.array(g["cores"], float), g["idx"]) == g["expect"]


def test_reconstruct_outer_S75(ora):
    g = GOLD["reconstruct_outer"]
    A = ora.tt_full(g["dims"], g["ranks"], np.array(g["cores"], float))
    assert A.tolist() == g["expect"]
    Af = ora.tt_full_f32(g["dims"], g["ranks"], np.array(g["cores"], float))
    assert Af.tolist() == g["expect"]


def _einsum_full(dims, ranks, cores):
    cs = ni.full_ranks(ranks)
    parts, off = [], 0
    for l in range(len(dims)):
        sz = cs[l] * dims[l] * cs[l + 1]
        parts.append(cores[off:off + sz].reshape(cs[l], dims[l], cs[l + 1]))
        off += sz
    A = parts[0]
    for G in parts[1:]:
        A = np.tensordot(A, G, axes=([A.ndim - 1], [0]))
    return A.reshape(dims)


@pytest.mark.parametrize("dims,ranks", [([5, 4, 5, 6], [4, 3, 2]), ([3, 4], [2]), ([2, 3, 2, 3, 2], [2, 3, 3, 2]),
                                        ([6] * 4, [5, 5, 5])])
def test_tt_full_vs_einsum_and_eq2(ora, dims, ranks):
    cores = ni.make_cores(dims, ranks, seed=1)
    A = ora.tt_full(dims, ranks, cores)
    B = _einsum_full(dims, ranks, cores)
    assert np.allclose(A, B, rtol=1e-13, atol=0)
    rng = np.random.default_rng(0)
    for _ in range(40):
        idx = [int(rng.integers(0, n)) for n in dims]
        e = ora.tt_element(dims, ranks, cores, idx)
        assert abs(e - A[tuple(idx)]) <= 1e-12 * abs(A[tuple(idx)])


def test_tt_full_f32_split_and_noise(ora):
    dims, ranks = [4, 3, 5, 2, 3], [2, 3, 2, 2]
    cores = ni.make_cores(dims, ranks, seed=2)
    A = _einsum_full(dims, ranks, cores)
    Af = ora.tt_full_f32(dims, ranks, cores)
    assert Af.dtype == np.float32
    # rounded once from the fp64 value: within half an ulp (+ fp64 slop)
    assert np.all(np.abs(Af.astype(np.float64) - A) <= np.spacing(Af).astype(np.float64) * 0.5 + 1e-12 * np.abs(A))
    An = ora.tt_full_f32(dims, ranks, cores, noise_amp=0.25, seed=9, noise_stream=0x300)
    u = ni.uniform(A.size, 9, 0x300).reshape(dims)
    expect = A + 0.25 * u
    assert np.all(np.abs(An.astype(np.float64) - expect) <= np.spacing(An).astype(np.float64) * 0.5 + 1e-12 * expect)


def test_tt_rank1_is_outer_product(ora):
    dims = [3, 4, 2]
    cores = ni.make_cores(dims, [1, 1], seed=4)
    a, b, c = cores[:3], cores[3:7], cores[7:]
    A = ora.tt_full(dims, [1, 1], cores)
    assert np.allclose(A, np.einsum("i,j,k->ijk", a, b, c), rtol=1e-15)


def test_rel_error_examples(ora):
    for g in GOLD["rel_error"]:
        a = np.array(g["a"], float)
        b = np.array(g["b"], float)
        assert ora.rel_error(a, b) == pytest.approx(g["expect"], abs=1e-15)
        assert ora.rel_error(a.astype(np.float32), b) == pytest.approx(g["expect"], abs=1e-15)
    assert ora.rel_error(np.zeros(3), np.ones(3)) == -1.0  # degenerate: ||A|| = 0
    # scale invariance
    rng = np.random.default_rng(3)
    a, b = rng.random(50), rng.random(50)
    assert ora.rel_error(a, b) == pytest.approx(ora.rel_error(4 * a, 4 * b), rel=1e-15)


def test_compression_ratio_examples(ora):
    for g in GOLD["compression_ratio"]:
        expect = Fraction(g["expect_num"], g["expect_den"])
        assert ora.compression_ratio(g["dims"], g["ranks"]) == pytest.approx(float(expect), rel=1e-15)


def test_tt_rel_error_matches_materialised(ora):
    dims, ranks = [5, 4, 5, 6], [4, 3, 2]
    cores = ni.make_cores(dims, ranks, seed=0)
    A = ora.tt_full_f32(dims, ranks, cores, noise_amp=0.3, seed=1)
    cores2 = ni.make_cores(dims, ranks, seed=5)
    B = ora.tt_full(dims, ranks, cores2)
    direct = np.sqrt(((A.astype(np.float64) - B) ** 2).sum() / (A.astype(np.float64) ** 2).sum())
    assert ora.tt_rel_error(A, ranks, cores2) == pytest.approx(direct, rel=1e-12)
    assert ora.rel_error(A, B) == pytest.approx(direct, rel=1e-12)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_tt_rel_error_split_matches(ora, k):
    dims, ranks = [5, 4, 5, 6], [4, 3, 2]
    A = ora.tt_full_f32(dims, ranks, ni.make_cores(dims, ranks, seed=0), noise_amp=0.3, seed=1)
    cores2 = ni.make_cores(dims, ranks, seed=5)
    assert ora.tt_rel_error_split(A, ranks, cores2, k) == pytest.approx(ora.tt_rel_error(A, ranks, cores2), rel=1e-12)


def test_core_offsets(ora):
    dims, ranks = [6] * 10, [5] * 9
    assert ora.core_offset(dims, ranks, 1) == 0
    assert ora.core_offset(dims, ranks, 2) == 30
    assert ora.core_offset(dims, ranks, 3) == 30 + 150
    assert ora.cores_size(dims, ranks) == 30 + 8 * 150 + 30 == 1260
    assert ora.cores_size([32] * 6, [8] * 5) == 256 + 4 * 2048 + 256 == 8704
    assert ora.cores_size([5, 4, 5, 6], [4, 3, 2]) == 110
