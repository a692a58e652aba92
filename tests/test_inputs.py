"""The seeded input generators (ntt_inputs; no method arithmetic): make_cores_decay scales
make_cores' entries by rho^(a + b), and its trains have the graded spectra the eps sweeps need
(checked against numpy's SVD of an unfolding built by the oracle's Eq. 1)."""
import numpy as np

import ntt_inputs as ni


def test_make_cores_decay_is_a_scaling_of_make_cores():
    dims, ranks = [4, 5, 6, 3], [3, 4, 2]
    c = ni.make_cores(dims, ranks, 7)
    assert np.array_equal(ni.make_cores_decay(dims, ranks, 1.0, 7), c)
    d = ni.make_cores_decay(dims, ranks, 0.5, 7)
    fr = [1, *ranks, 1]
    o = 0
    for l in range(len(dims)):
        a, n, b = fr[l], dims[l], fr[l + 1]
        G, Gd = c[o:o + a * n * b].reshape(a, n, b), d[o:o + a * n * b].reshape(a, n, b)
        for i in range(a):
            for k in range(b):
                assert np.array_equal(Gd[i, :, k], G[i, :, k] * 0.5 ** (i + k))  # powers of 2: exact
        o += a * n * b


def test_make_cores_decay_spectrum_is_graded(ora):
    """U[0,1) trains: one dominant direction then a flat rest; rho < 1: geometric decay, so the
    eps-driven rank rule (Alg. 2 l.5-6) picks different ranks for different eps."""
    dims, ranks = [16, 16, 16], [8, 8]
    flat = ora.tt_full(dims, ranks, ni.make_cores(dims, ranks, 0)).reshape(16, -1)
    dec = ora.tt_full(dims, ranks, ni.make_cores_decay(dims, ranks, 0.6, 0)).reshape(16, -1)
    sf = np.linalg.svd(flat, compute_uv=False)
    sd = np.linalg.svd(dec, compute_uv=False)
    # the flat train's 2nd..8th singular values stay within 10x of each other
    assert sf[1] / sf[7] < 10
    # the graded train's decay by more than 100x over the same range
    assert sd[1] / sd[7] > 100
    ranks_at = {eps: ora.svd_tail_rank(dec, eps) for eps in (0.1, 0.03, 0.01, 0.003)}
    assert len(set(ranks_at.values())) >= 3, ranks_at
