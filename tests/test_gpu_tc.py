"""GPU parity of the tensor-core (tcgen05 kind::tf32, 3xTF32) 2-pass MU path
(mu_tc.cu; tall / square X, BASELINE configs 2 and 5) against the CPU oracle.

Tolerance: readings R14 (north_star: factors within 1e-4 relative after 10
iterations).  The path must actually run (profile classes 6 / 7 launched).
"""
import numpy as np
import pytest

import ntt_inputs as ni

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def h():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2008_01340_b200 as P
    return P.Handle(0)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def rel(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    return (np.linalg.norm(got - ref) / np.linalg.norm(ref), np.abs(got - ref).max() / np.abs(ref).max())


def inputs(m, n, r, seed, kind="rand"):
    rng = np.random.default_rng(seed)
    if kind == "lowrank":  # X = W0 H0 + noise, the BASELINE configs 2 / 5 recipe shape
        X = (rng.random((m, r)) @ rng.random((r, n)) + 0.01 * rng.random((m, n))).astype(np.float32)
    else:
        X = (rng.random((m, n)) * 4).astype(np.float32)
    W0 = ni.uniform(m * r, seed, 0x202).reshape(m, r).astype(np.float32)
    H0 = ni.uniform(r * n, seed, 0x203).reshape(r, n).astype(np.float32)
    return X, W0, H0


TC_CASES = [
    # m, n, r, iters, kind
    (512, 1024, 16, 1, "rand"),
    (512, 1000, 16, 10, "rand"),
    (1000, 776, 32, 10, "rand"),
    (2048, 3000, 32, 10, "lowrank"),
    (300, 4100, 12, 10, "rand"),
    (257, 260, 5, 10, "rand"),
    (4096, 4096, 16, 3, "lowrank"),   # config 2 shape
    (8192, 2048, 32, 2, "lowrank"),   # config 5-like (tall)
]


@pytest.mark.parametrize("m,n,r,iters,kind", TC_CASES)
def test_tc_mu_parity(h, ora, m, n, r, iters, kind):
    X, W0, H0 = inputs(m, n, r, m + 3 * n + r, kind)
    Xd, Wd, Hd = dev(X), dev(W0), dev(H0)
    h.ntt_profile_enable(True)
    h.ntt_nmf_mu(Xd, m, n, n, r, iters, 1e-16, Wd, Hd)
    k6, _, _ = h.ntt_profile_get(6)
    k7, _, _ = h.ntt_profile_get(7)
    h.ntt_profile_enable(False)
    assert k6 == iters and k7 == iters, "tensor-core path not taken"
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), iters, eps=1e-16)
    Wg, Hg = host(Wd), host(Hd)
    for name, g, o in (("W", Wg, Wo), ("H", Hg, Ho)):
        fro, mx = rel(g, o)
        assert np.all(np.isfinite(g)) and np.all(g >= 0), name
        assert fro <= TOL and mx <= TOL, f"{name} {m}x{n} r{r}: rel fro {fro:.3e}, rel max {mx:.3e}"


def test_tc_scale_invariance_and_determinism(h):
    """X -> 8X gives W -> 8W and H unchanged bit for bit (the hi/lo split commutes with
    powers of two); repeated runs are bit-identical (fixed-order split-K sums)."""
    m, n, r = 1024, 2048, 32
    X, W0, H0 = inputs(m, n, r, 11)
    outs = []
    for scale in (1.0, 8.0, 1.0):
        Wd, Hd = dev(W0), dev(H0)
        h.ntt_nmf_mu(dev(X * np.float32(scale)), m, n, n, r, 4, 0.0, Wd, Hd)
        outs.append((host(Wd), host(Hd)))
    assert np.array_equal(outs[0][0], outs[2][0]) and np.array_equal(outs[0][1], outs[2][1])
    assert np.array_equal(outs[1][0], 8 * outs[0][0])
    assert np.array_equal(outs[1][1], outs[0][1])


def test_tc_leading_dimension(h, ora):
    m, n, r, ldx = 600, 900, 16, 1000
    X, W0, H0 = inputs(m, ldx, r, 5)
    H0 = np.ascontiguousarray(H0[:, :n])
    Xd, Wd, Hd = dev(X), dev(W0), dev(H0)
    h.ntt_nmf_mu(Xd, m, n, ldx, r, 5, 1e-16, Wd, Hd)
    Wo, Ho = ora.nmf_mu(np.ascontiguousarray(X[:, :n]), W0.astype(np.float64), H0.astype(np.float64), 5)
    for g, o in ((host(Wd), Wo), (host(Hd), Ho)):
        fro, mx = rel(g, o)
        assert fro <= TOL and mx <= TOL, (fro, mx)


@pytest.mark.parametrize("variant", ["0", "1"])
@pytest.mark.parametrize("m,n,r,wide", [(1000, 776, 32, False), (512, 1024, 16, True), (2048, 1536, 24, True)])
def test_tc_variants_parity(h, ora, variant, m, n, r, wide):
    """Both tensor-core variants (NTT_TC16=0: 3xTF32, =1: fp16x2 with power-of-two
    scales) match the oracle; `wide` spreads X over ~9 decades (row and column
    scales 1e-4 .. 1e4) to exercise the fp16 scaling and subnormal floor."""
    import os
    X, W0, H0 = inputs(m, n, r, 17 + m)
    if wide:
        rng = np.random.default_rng(5)
        X = (X * 10.0 ** rng.uniform(-2, 2, (m, 1)) * 10.0 ** rng.uniform(-2, 2, (1, n))).astype(np.float32)
    os.environ["NTT_TC16"] = variant
    try:
        Xd, Wd, Hd = dev(X), dev(W0), dev(H0)
        h.ntt_nmf_mu(Xd, m, n, n, r, 8, 1e-16, Wd, Hd)
        Wg, Hg = host(Wd), host(Hd)
    finally:
        os.environ.pop("NTT_TC16", None)
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), 8, eps=1e-16)
    for name, g, o in (("W", Wg, Wo), ("H", Hg, Ho)):
        fro, mx = rel(g, o)
        assert np.all(np.isfinite(g)) and np.all(g >= 0), name
        assert fro <= TOL and mx <= TOL, f"{name} variant {variant}: rel fro {fro:.3e}, rel max {mx:.3e}"
