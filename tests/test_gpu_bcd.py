"""GPU parity of the BCD NMF (Alg. 3; readings R22-R27; SURVEY s.8(f) f1)
against oracle.nmf_bcd.

Both sides start from the same fp32 inputs; the GPU stores W, H in fp32 (fp64 sums and
r x r matrices), the oracle is fp64 throughout.  Tolerances: factors 1e-4 relative to their
max entry, accepted objective 1e-5 relative, over a bounded number of iterations (the
accept / correct branch of l.17 is decided by the objective; the inputs keep clear
decreases in that window, so both sides take the same branches — checked)."""
import numpy as np
import pytest

import ntt_inputs as ni

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def h():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2008_01340_b200 as P
    return P.Handle(0)


def case(m, n, r, seed, lowrank=0):
    rng = np.random.default_rng(seed)
    if lowrank:
        X = rng.random((m, lowrank)) @ rng.random((lowrank, n)) + 0.01 * rng.random((m, n))
    else:
        X = rng.random((m, n))
    X = X.astype(np.float32)
    W0 = ni.uniform(m * r, seed, ni.stream_w(1)).reshape(m, r).astype(np.float32)
    H0 = ni.uniform(r * n, seed, ni.stream_h(1)).reshape(r, n).astype(np.float32)
    return X, W0, H0


def run_gpu(h, X, W0, H0, iters, delta=0.9999):
    m, n = X.shape
    r = W0.shape[1]
    Xd = torch.from_numpy(X.ravel()).cuda()
    Wd = torch.from_numpy(W0.ravel().copy()).cuda()
    Hd = torch.from_numpy(H0.ravel().copy()).cuda()
    tr = h.ntt_nmf_bcd(Xd, m, n, n, r, iters, Wd, Hd, delta=delta, trace=True)
    return Wd.cpu().numpy().reshape(m, r), Hd.cpu().numpy().reshape(r, n), np.array(tr)


def branches(tr, obj0):
    prev = np.concatenate([[obj0], tr[:-1]])
    return tr < prev        # True = accepted (extrapolation), False = correction


@pytest.mark.parametrize("m,n,r,iters,lr", [
    (40, 300, 4, 15, 0), (257, 1000, 8, 15, 0), (100, 2000, 16, 12, 6), (513, 777, 32, 10, 0),
    (3000, 64, 5, 15, 3), (1, 50, 1, 8, 0), (7, 7, 7, 10, 0),
    # m <= 40 and n % 32 == 0: the one-pass kernel forms H_m = a H_prev - b H_prev2 itself
    # (BS_FOLD); 15 iterations keep several accepted extrapolations in the window
    (32, 4096, 8, 15, 0), (6, 2048, 5, 15, 0), (24, 1024, 4, 12, 3),
    # 40 < m <= 256: one-pass k_fused_c; at n = 2^15 its 2-per-SM partials are pre-summed across
    # the GPU before the one-CTA post kernel
    (256, 32768, 8, 10, 0), (64, 8192, 8, 10, 4),
    # 9 <= r <= 16 at 40 < m <= 256: k_fused_c's rank-16 class in BCD mode (one CTA of 8 consumer
    # warps for m > 128)
    (200, 4096, 10, 10, 0), (256, 2048, 16, 8, 0), (72, 1000, 12, 10, 5)])
def test_bcd_parity(h, ora, m, n, r, iters, lr):
    X, W0, H0 = case(m, n, r, m * 7 + n + r, lr)
    Wg, Hg, trg = run_gpu(h, X, W0, H0, iters)
    Wo, Ho, tro = ora.nmf_bcd(X.astype(np.float64), W0, H0, iters, trace=True)
    obj0 = 0.5 * float(np.sum(X.astype(np.float64) ** 2))
    assert np.array_equal(branches(trg, obj0), branches(tro, obj0))
    # the GPU evaluates the objective by the Gram identity from X H^T, whose contraction runs
    # in fp32 chunks (FFMA) or fp16x2 parts with fp32 tensor-core accumulation (m, n >= 256):
    # a ~1e-6-relative error in <W, X H^T> scales with ||X||^2 = 2 obj0, hence the
    # ||X||^2-relative term (R25).
    assert np.abs(trg - tro).max() <= 1e-5 * tro.max() + 1e-5 * obj0
    assert np.abs(Wg - Wo).max() <= 1e-4 * np.abs(Wo).max()
    assert np.abs(Hg - Ho).max() <= 1e-4 * np.abs(Ho).max()
    assert Wg.min() >= 0 and Hg.min() >= 0


FORCED = (2, 3, 6)   # iterations forced onto the correction branch (two in a row, then one more)


@pytest.mark.parametrize("m,n,r,lr", [
    (32, 4096, 8, 0),     # one pass, H_m folded inside k_fused (BS_FOLD)
    (9, 40, 4, 0),        # one pass k_fused, H_m materialised (no fold: n % 32 != 0)
    (256, 32768, 8, 0),   # one pass k_fused_c, GPU-wide partial pre-sum
    (64, 8192, 8, 4),     # one pass k_fused_c
    (300, 512, 16, 0),    # fp16x2 tensor-core passes, large-W kernels
    (100, 2000, 16, 6),   # one pass k_fused_c, rank-16 class; one-CTA W side / post kernels
    (200, 4096, 12, 0),   # one pass k_fused_c, rank-16 class with 8 consumer warps
    (3000, 64, 5, 3),     # FFMA passes, large-W kernels
    (7, 7, 7, 0)])        # generic small case
def test_bcd_forced_correction_parity(h, ora, m, n, r, lr):
    """Alg. 3 l.17-20 (reading R26) on every BCD path: the hook forces the
    correction branch at iterations 2, 3 and 6; GPU and oracle (same hook) must agree on the
    branches, the accepted objectives and the factors.  After a correction the returned
    factors are the last accepted ones, t restarts at 1 (w = 0 in the next accepted step)
    and P, Q come from the rescaled H_prev (no pass over X)."""
    iters = 10
    X, W0, H0 = case(m, n, r, m * 3 + n + r, lr)
    h.ntt_debug_bcd_force_correct(FORCED)
    try:
        Wg, Hg, trg = run_gpu(h, X, W0, H0, iters)
    finally:
        h.ntt_debug_bcd_force_correct(())
    log = []
    Wo, Ho, tro = ora.nmf_bcd(X.astype(np.float64), W0, H0, iters, trace=True, log=log,
                              force_correct=set(FORCED))
    obj0 = 0.5 * float(np.sum(X.astype(np.float64) ** 2))
    acc_o = np.array([e["accepted"] for e in log])
    assert (~acc_o).sum() >= len(FORCED)
    assert np.array_equal(branches(trg, obj0), acc_o)
    # a forced correction leaves the accepted objective where it was
    for i in FORCED:
        assert trg[i] == (trg[i - 1] if i else obj0)
    assert np.abs(trg - tro).max() <= 1e-5 * tro.max() + 1e-5 * obj0
    assert np.abs(Wg - Wo).max() <= 1e-4 * np.abs(Wo).max()
    assert np.abs(Hg - Ho).max() <= 1e-4 * np.abs(Ho).max()


# (m, n, r, seed, kind, iterations): inputs on which the extrapolation overshoots by itself,
# run to two iterations past the second correction; every objective change up to there is
# >= 1.6e-6 * 1/2 ||X||^2, far above the fp32 resolution of the GPU's Gram-identity
# objective (~1e-7 of it; R25), so the branch decisions are well posed on both sides
NATURAL = [(7, 64, 3, 11, "scaled", 52), (7, 64, 3, 10, "colscaled", 63)]


@pytest.mark.parametrize("m,n,r,seed,kind,iters", NATURAL)
def test_bcd_natural_correction_parity(h, ora, m, n, r, seed, kind, iters):
    """Inputs on which the extrapolation overshoots by itself (ntt_inputs.bcd_overshoot_matrix:
    row / column scales over three decades): the oracle takes >= 2 corrections (asserted), and
    the GPU takes the same branches with factors within 1e-4."""
    import ntt_inputs as ni
    X = ni.bcd_overshoot_matrix(m, n, r, seed, kind)
    W0 = ni.uniform(m * r, seed, ni.stream_w(1)).reshape(m, r).astype(np.float32)
    H0 = ni.uniform(r * n, seed, ni.stream_h(1)).reshape(r, n).astype(np.float32)
    Wg, Hg, trg = run_gpu(h, X, W0, H0, iters)
    log = []
    Wo, Ho, tro = ora.nmf_bcd(X.astype(np.float64), W0, H0, iters, trace=True, log=log)
    obj0 = 0.5 * float(np.sum(X.astype(np.float64) ** 2))
    corr = [e["it"] for e in log if not e["accepted"]]
    assert len(corr) >= 2
    assert np.array_equal(branches(trg, obj0), np.array([e["accepted"] for e in log]))
    assert np.abs(trg - tro).max() <= 1e-5 * tro.max() + 1e-5 * obj0
    assert np.abs(Wg - Wo).max() <= 1e-4 * np.abs(Wo).max()
    assert np.abs(Hg - Ho).max() <= 1e-4 * np.abs(Ho).max()


def test_bcd_zero_iterations_rescales(h, ora):
    X, W0, H0 = case(30, 70, 3, 1)
    Wg, Hg, _ = run_gpu(h, X, W0, H0, 0)
    Wo, Ho = ora.nmf_bcd(X.astype(np.float64), W0, H0, 0)
    assert np.allclose(Wg, Wo, rtol=1e-6, atol=0) and np.allclose(Hg, Ho, rtol=1e-6, atol=0)
    nx = np.linalg.norm(X.astype(np.float64))
    assert abs(np.linalg.norm(Wg.astype(np.float64)) - np.sqrt(nx)) <= 1e-6 * np.sqrt(nx)


def test_bcd_delta_zero(h, ora):
    """delta = 0 switches extrapolation off (w_W = w_H = 0): plain prox-linear BCD."""
    X, W0, H0 = case(64, 200, 6, 5)
    Wg, Hg, trg = run_gpu(h, X, W0, H0, 12, delta=0.0)
    Wo, Ho, tro = ora.nmf_bcd(X.astype(np.float64), W0, H0, 12, delta=0.0, trace=True)
    assert np.abs(trg - tro).max() <= 1e-5 * tro.max() + 1e-5 * 0.5 * float(np.sum(X.astype(np.float64) ** 2))
    assert np.abs(Wg - Wo).max() <= 1e-4 * np.abs(Wo).max()
    assert np.abs(Hg - Ho).max() <= 1e-4 * np.abs(Ho).max()


def test_bcd_errors(h):
    import paper_2008_01340_b200 as P
    X = torch.rand(20 * 40, device="cuda")
    W = torch.rand(20 * 33, device="cuda")
    H = torch.rand(33 * 40, device="cuda")
    with pytest.raises(P.NttError):
        h.ntt_nmf_bcd(X, 20, 40, 40, 33, 5, W, H)          # r > 32
    with pytest.raises(P.NttError):
        h.ntt_nmf_bcd(X, 20, 40, 40, 4, 5, W, H, delta=1.0)
    Z = torch.zeros(20 * 40, device="cuda")
    with pytest.raises(P.NttError):
        h.ntt_nmf_bcd(Z, 20, 40, 40, 4, 5, W, H)            # ||X|| = 0
    with pytest.raises(P.NttError, match="W0"):
        h.ntt_nmf_bcd(X, 20, 40, 40, 4, 5, torch.zeros(20 * 4, device="cuda"), H)   # ||W0|| = 0 (l.2)
    with pytest.raises(P.NttError, match="H0"):
        h.ntt_nmf_bcd(X, 20, 40, 40, 4, 5, W, torch.zeros(4 * 40, device="cuda"))   # ||H0|| = 0


def test_bcd_fullsize_properties(h):
    """Config-2 size (4096 x 4096, r = 16): accepted objective non-increasing, factors
    non-negative, trace = 1/2 ||X - W H||_F^2 of the returned factors, and lower error
    than the same number of MU iterations from the same start (the paper's claim)."""
    m = n = 4096
    r, iters = 16, 40
    g = torch.Generator(device="cuda").manual_seed(2)
    Wt = torch.rand(m, r, device="cuda", generator=g)
    Ht = torch.rand(r, n, device="cuda", generator=g)
    X = (Wt @ Ht + 0.1 * torch.rand(m, n, device="cuda", generator=g)).contiguous()
    W0 = torch.rand(m * r, device="cuda", generator=g)
    H0 = torch.rand(r * n, device="cuda", generator=g)
    W, H = W0.clone(), H0.clone()
    tr = np.array(h.ntt_nmf_bcd(X.view(-1), m, n, n, r, iters, W, H, trace=True))
    assert np.all(np.diff(tr) <= 0) and W.min() >= 0 and H.min() >= 0
    Xd = X.double()
    res = 0.5 * float(((Xd - W.view(m, r).double() @ H.view(r, n).double()) ** 2).sum())
    obj0 = 0.5 * float((Xd ** 2).sum())
    assert abs(res - tr[-1]) <= 1e-5 * obj0      # Gram-identity objective (R25)
    Wm, Hm = W0.clone(), H0.clone()
    h.ntt_nmf_mu(X.view(-1), m, n, n, r, iters, 1e-16, Wm, Hm)
    res_mu = 0.5 * float(((Xd - Wm.view(m, r).double() @ Hm.view(r, n).double()) ** 2).sum())
    assert res < res_mu


@pytest.mark.parametrize("dims,ranks,iters", [((5, 4, 5, 6), (4, 3, 2), 10), ((6, 6, 6, 6, 6), (5, 5, 5, 5), 8),
                                              ((300, 20, 40), (12, 9), 6)])
def test_ntt_bcd_sweep_parity(h, ora, dims, ranks, iters):
    """nTT with BCD at every step (Alg. 2 + Alg. 3) against oracle.ntt_decompose_bcd: cores
    1e-4 relative per core (R14), Eq. 3 error within 1e-3 (R15)."""
    import paper_2008_01340_b200 as P
    rng = np.random.default_rng(sum(dims))
    A = (ora.tt_full(list(dims), list(ranks), rng.random(ora.cores_size(list(dims), list(ranks))))
         + 0.01 * rng.random(dims)).astype(np.float32)
    cores = torch.empty(P.cores_size(list(dims), list(ranks)), device="cuda")
    err = h.ntt_decompose_bcd(torch.from_numpy(A.ravel()).cuda(), list(dims), list(ranks), iters, 0, cores,
                              want_error=True)
    co = ora.ntt_decompose_bcd(A, list(ranks), iters)
    cg = cores.cpu().numpy().astype(np.float64)
    for Gg, Go in zip(ora.unpack_cores(list(dims), list(ranks), cg), ora.unpack_cores(list(dims), list(ranks), co)):
        assert np.abs(Gg - Go).max() <= 1e-4 * np.abs(Go).max()
    e_ora = ora.rel_error(A, ora.tt_full(list(dims), list(ranks), co))
    assert abs(err - e_ora) <= 1e-3 * e_ora + 1e-6


def test_ntt_bcd_sweep_host_buffers_and_errors(h, ora):
    """Host A / host cores through ntt_decompose_bcd (staged by the library) equal the device
    call bit for bit; ranks > 32 and delta outside [0, 1) are rejected."""
    import paper_2008_01340_b200 as P
    dims, ranks = [5, 4, 5, 6], [4, 3, 2]
    rng = np.random.default_rng(3)
    A = rng.random(dims).astype(np.float32)
    cd = torch.empty(P.cores_size(dims, ranks), device="cuda")
    e_dev = h.ntt_decompose_bcd(torch.from_numpy(A.ravel()).cuda(), dims, ranks, 5, 0, cd, want_error=True)
    ch = np.empty(P.cores_size(dims, ranks), dtype=np.float32)
    e_host = h.ntt_decompose_bcd(np.ascontiguousarray(A.ravel()), dims, ranks, 5, 0, ch, want_error=True)
    assert np.array_equal(cd.cpu().numpy(), ch) and e_dev == e_host
    with pytest.raises(P.NttError):
        h.ntt_decompose_bcd(torch.from_numpy(A.ravel()).cuda(), dims, [4, 33, 2], 5, 0, cd)
    with pytest.raises(P.NttError):
        h.ntt_decompose_bcd(torch.from_numpy(A.ravel()).cuda(), dims, ranks, 5, 0, cd, delta=1.5)
