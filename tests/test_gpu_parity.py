"""GPU parity: libntt's sm_100a kernels (through the C ABI) vs the CPU oracle.

Tolerances (BASELINE north_star, readings R14/R15, DESIGN.md s.6):
  factors / cores after <= 10 iterations (and after the full config-1 run):
      ||G_gpu - G_ora||_F <= 1e-4 ||G_ora||_F  and  max|G_gpu - G_ora| <= 1e-4 max|G_ora|
  final relative reconstruction error:  |e_gpu - e_ora| <= 1e-3 e_ora + 1e-6
  RNG / init: bit exact.
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


def assert_close_factor(got, ref, tol=TOL, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape
    assert np.all(np.isfinite(got)), what
    fro = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    mx = np.abs(got - ref).max() / np.abs(ref).max()
    assert fro <= tol and mx <= tol, f"{what}: rel fro {fro:.3e}, rel max {mx:.3e}"


# ------------------------------------------------------------------- RNG ------
@pytest.mark.parametrize("seed,stream,off", [(0, 0x203, 0), (12345, 0x201, 7), (2**63 + 1, 0x300, 2**33)])
def test_fill_uniform_bit_exact(h, ora, seed, stream, off):
    n = 300_001
    t = torch.empty(n, dtype=torch.float32, device="cuda")
    h.ntt_fill_uniform(t, n, seed, stream, off)
    got = host(t).astype(np.float64)
    assert np.array_equal(got, ni.uniform(n, seed, stream, off))
    idx = [0, 1, 17, n - 1]
    assert [got[i] for i in idx] == [ora.fill_uniform(1, seed, stream, off + i)[0] for i in idx]


@pytest.mark.parametrize("shift,n", [(1, 100_003), (2, 7), (0, 3), (0, 1 << 20)])
def test_fill_uniform_alignment(h, shift, n):
    """128-bit store path (16-byte aligned, ragged count) and the scalar path (misaligned start)."""
    t = torch.zeros(n + 8, dtype=torch.float32, device="cuda")
    h.ntt_fill_uniform(t[shift:], n, 11, 0x207, 5)
    got = host(t).astype(np.float64)
    assert np.array_equal(got[shift:shift + n], ni.uniform(n, 11, 0x207, 5))
    assert not got[:shift].any() and not got[shift + n:].any()


def test_fill_uniform_host_pointer(h):
    a = np.empty(1000, np.float32)
    h.ntt_fill_uniform(a, 1000, 3, 0x205, 0)
    assert np.array_equal(a.astype(np.float64), ni.uniform(1000, 3, 0x205))


# ---------------------------------------------------------------- MU NMF -----
MU_CASES = [
    # m, n, r, iters  -- short-wide (1-pass), ragged tails, tall / square (2-pass), r up to 32
    (5, 120, 4, 10),
    (16, 30, 3, 10),
    (32, 5003, 8, 10),
    (6, 10001, 5, 10),
    (30, 4097, 5, 10),
    (256, 2051, 8, 10),
    (128, 700, 16, 10),
    (700, 90, 3, 10),
    (300, 257, 32, 6),
    (1, 50, 1, 10),
    (40, 1, 1, 10),
    # generic two-pass with the split-K H pass (few column tiles, many rows; the 500 GB tensor's
    # step 3 shape at r 40, and r 20 with n < 256 so the tensor-core path does not take it)
    (15360, 64, 40, 6),
    (3000, 200, 20, 10),
    # fused 1-pass TMA kernel (m <= 40, r <= 8, n % 4 == 0): every (R, UX) class, ragged last tile
    (32, 5004, 8, 10),
    (32, 1 << 16, 8, 10),
    (6, 10004, 5, 10),
    (30, 4100, 5, 10),
    (40, 1000, 8, 10),
    (16, 28, 3, 10),
    (8, 132, 2, 10),
    (15, 388, 4, 10),
    (5, 120, 1, 10),
    (24, 640, 7, 10),
    # fused CTA-cooperative variant (40 < m <= 256, r <= 8 padded to 8)
    (256, 2052, 8, 10),
    (256, 1 << 15, 8, 10),
    (64, 4096, 8, 10),
    (100, 1000, 5, 10),
    (200, 4100, 3, 10),
    (41, 260, 8, 10),
    # tensor-core one-pass kernels: k_fused_m (16 < m <= 32, n % 32 == 0; ragged 128-column tiles,
    # n < 128) and k_fused_c's X16 cache with row blocks beyond m (persistent, 30 passes)
    (17, 4096, 8, 10),
    (32, 4128, 3, 10),
    (20, 96, 6, 10),
    (30, 7776, 5, 12),
    (72, 8192, 8, 30),
    (200, 16384, 8, 30),
    (136, 2080, 6, 30),
    # k_fused_c's rank-16 class (9 <= r <= 16; the paper's 256^4 ranks 10): persistent + X16
    (256, 16384, 10, 30),
    (256, 4100, 12, 10),
    (100, 8192, 16, 20),
    (64, 1000, 9, 10),
]


@pytest.mark.parametrize("m,n,r", [(32, 4096, 5), (256, 1024, 5), (6, 1000, 3)])
def test_nmf_mu_eps_zero_padded_rank(h, ora, m, n, r):
    """eps = 0 with r < padded kernel rank must not produce 0/0 in the padding."""
    X, W0, H0 = _mu_inputs(m, n, r, 9)
    X += 0.5
    Xd, Wd, Hd = dev(X), dev(W0), dev(H0)
    h.ntt_nmf_mu(Xd, m, n, n, r, 6, 0.0, Wd, Hd)
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), 6, eps=0.0)
    assert_close_factor(host(Wd), Wo, what="W eps0")
    assert_close_factor(host(Hd), Ho, what="H eps0")


def _mu_inputs(m, n, r, seed):
    rng = np.random.default_rng(seed)
    X = (rng.random((m, n)) * 4).astype(np.float32)
    W0 = ni.uniform(m * r, seed, 0x202).reshape(m, r).astype(np.float32)
    H0 = ni.uniform(r * n, seed, 0x203).reshape(r, n).astype(np.float32)
    return X, W0, H0


@pytest.mark.parametrize("m,n,r,iters", MU_CASES)
def test_nmf_mu_parity(h, ora, m, n, r, iters, monkeypatch):
    # the grid-wide / tiny / two-pass kernels: cluster mode (tested below) would take the
    # mid-size shapes here, so it is switched off for this list
    monkeypatch.setenv("NTT_NO_CLUSTER", "1")
    assert h.mu_path(m, n, r) != 2
    X, W0, H0 = _mu_inputs(m, n, r, m * 7 + n)
    Xd, Wd, Hd = dev(X), dev(W0), dev(H0)
    h.ntt_nmf_mu(Xd, m, n, n, r, iters, 1e-16, Wd, Hd)
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), iters, eps=1e-16)
    assert_close_factor(host(Wd), Wo, what=f"W {m}x{n} r{r}")
    assert_close_factor(host(Hd), Ho, what=f"H {m}x{n} r{r}")
    assert np.all(host(Wd) >= 0) and np.all(host(Hd) >= 0)


# cluster mode (mu_cluster.cu): X in the distributed shared memory of one thread-block cluster.
# Config 3 steps 4-5 and config 4 steps 5-6 shapes, ragged column / row ownership across the
# CTAs (incl. CTAs that own no W row), both rank classes (RK = 8, 16), 1..16-CTA clusters.
CLU_CASES = [
    (256, 1024, 8, 10),
    (256, 40, 8, 10),
    (30, 1296, 5, 12),
    (256, 1000, 8, 10),
    (100, 1000, 5, 10),
    (200, 333, 16, 10),
    (41, 600, 8, 10),
    (128, 700, 16, 10),
    (64, 300, 9, 30),
    (30, 2000, 5, 10),
    (64, 1024, 16, 10),
    (8, 2000, 3, 10),
]


@pytest.mark.parametrize("m,n,r,iters", CLU_CASES)
def test_nmf_mu_cluster_parity(h, ora, m, n, r, iters):
    assert h.mu_path(m, n, r) == 2, "shape should take cluster mode"
    X, W0, H0 = _mu_inputs(m, n, r, m * 5 + n)
    Xd, Wd, Hd = dev(X), dev(W0), dev(H0)
    h.ntt_nmf_mu(Xd, m, n, n, r, iters, 1e-16, Wd, Hd)
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), iters, eps=1e-16)
    W1, H1 = host(Wd), host(Hd)
    assert_close_factor(W1, Wo, what=f"W {m}x{n} r{r}")
    assert_close_factor(H1, Ho, what=f"H {m}x{n} r{r}")
    assert np.all(W1 >= 0) and np.all(H1 >= 0)
    # fixed-order sums: a second run is bit-identical
    Wd2, Hd2 = dev(W0), dev(H0)
    h.ntt_nmf_mu(Xd, m, n, n, r, iters, 1e-16, Wd2, Hd2)
    assert np.array_equal(host(Wd2), W1) and np.array_equal(host(Hd2), H1)


def test_nmf_mu_cluster_leading_dimension(h, ora):
    m, n, r, ldx = 256, 1000, 8, 1030
    X, W0, H0 = _mu_inputs(m, ldx, r, 6)
    H0 = np.ascontiguousarray(H0[:, :n])
    assert h.mu_path(m, n, r) == 2
    Xd, Wd, Hd = dev(X), dev(W0), dev(H0)
    h.ntt_nmf_mu(Xd, m, n, ldx, r, 8, 1e-16, Wd, Hd)
    Wo, Ho = ora.nmf_mu(np.ascontiguousarray(X[:, :n]), W0.astype(np.float64), H0.astype(np.float64), 8)
    assert_close_factor(host(Wd), Wo, what="W ldx")
    assert_close_factor(host(Hd), Ho, what="H ldx")


def test_nmf_mu_leading_dimension(h, ora):
    m, n, r, ldx = 20, 333, 4, 400
    X, W0, H0 = _mu_inputs(m, ldx, r, 5)
    H0 = np.ascontiguousarray(H0[:, :n])
    Xd, Wd, Hd = dev(X), dev(W0), dev(H0)
    h.ntt_nmf_mu(Xd, m, n, ldx, r, 8, 1e-16, Wd, Hd)
    Wo, Ho = ora.nmf_mu(np.ascontiguousarray(X[:, :n]), W0.astype(np.float64), H0.astype(np.float64), 8)
    assert_close_factor(host(Wd), Wo, what="W ldx")
    assert_close_factor(host(Hd), Ho, what="H ldx")


def test_nmf_mu_objective_trace_and_monotone(h, ora):
    m, n, r, iters = 24, 999, 4, 25
    X, W0, H0 = _mu_inputs(m, n, r, 1)
    Xd, Wd, Hd = dev(X), dev(W0), dev(H0)
    tr = np.array(h.ntt_nmf_mu(Xd, m, n, n, r, iters, 1e-16, Wd, Hd, trace=True))
    _, _, tro = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), iters, trace=True)
    assert np.allclose(tr, tro, rtol=1e-4)
    assert np.all(np.diff(tr) <= 1e-5 * tr[:-1])


def test_nmf_mu_host_pointers(h, ora):
    m, n, r = 12, 500, 3
    X, W0, H0 = _mu_inputs(m, n, r, 2)
    W, H = W0.copy(), H0.copy()
    h.ntt_nmf_mu(X, m, n, n, r, 5, 1e-16, W, H)
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), 5)
    assert_close_factor(W, Wo, what="W host")
    assert_close_factor(H, Ho, what="H host")


def test_nmf_mu_zero_iterations_is_identity(h):
    X, W0, H0 = _mu_inputs(8, 64, 2, 3)
    Wd, Hd = dev(W0), dev(H0)
    h.ntt_nmf_mu(dev(X), 8, 64, 64, 2, 0, 1e-16, Wd, Hd)
    assert np.array_equal(host(Wd), W0) and np.array_equal(host(Hd), H0)


@pytest.mark.parametrize("m,n,r", [(32, 4096, 8), (256, 2048, 8), (20, 999, 4)])
def test_nmf_mu_scale_invariance_and_determinism(h, m, n, r):
    """Metamorphic (no oracle): X -> 8X gives W -> 8W, H unchanged; repeat runs bit-identical."""
    X, W0, H0 = _mu_inputs(m, n, r, 4)
    outs = []
    for scale in (1.0, 8.0, 1.0):
        Wd, Hd = dev(W0), dev(H0)
        h.ntt_nmf_mu(dev(X * np.float32(scale)), m, n, n, r, 5, 0.0, Wd, Hd)
        outs.append((host(Wd), host(Hd)))
    assert np.array_equal(outs[0][0], outs[2][0]) and np.array_equal(outs[0][1], outs[2][1])
    assert np.array_equal(outs[1][0], 8 * outs[0][0])
    assert np.array_equal(outs[1][1], outs[0][1])


@pytest.mark.parametrize("bad", ["rank0", "rank_big", "ldx", "iters"])
def test_nmf_mu_rejects_bad_args(h, bad):
    import paper_2008_01340_b200 as P
    X, W0, H0 = _mu_inputs(8, 64, 2, 3)
    args = dict(m=8, n=64, ldx=64, r=2, iters=3)
    if bad == "rank0":
        args["r"] = 0
    elif bad == "rank_big":
        args["r"] = 9
    elif bad == "ldx":
        args["ldx"] = 10
    else:
        args["iters"] = -1
    with pytest.raises(P.NttError) as e:
        h.ntt_nmf_mu(dev(X), args["m"], args["n"], args["ldx"], args["r"], args["iters"], 1e-16, dev(W0), dev(H0))
    assert e.value.status == (3 if bad.startswith("rank") else 1)


# ----------------------------------------------------------------- nTT -------
def _tt_case(dims, ranks, seed=0, noise=0.0):
    import oracle
    cores = ni.make_cores(dims, ranks, seed)
    A = oracle.tt_full_f32(dims, ranks, cores, noise_amp=noise, seed=seed)
    return A


def _cores_check(dims, ranks, got, ref, tol=TOL):
    import oracle
    for l, (g, o) in enumerate(zip(oracle.unpack_cores(dims, ranks, got), oracle.unpack_cores(dims, ranks, ref))):
        assert_close_factor(g, o, tol, what=f"core {l + 1}")


NTT_CASES = [
    # dims, ranks, iters, noise
    ([5, 4, 5, 6], [4, 3, 2], 10, 0.0),      # config 1 shape at the 10-iteration parity point
    ([5, 4, 5, 6], [4, 3, 2], 200, 0.0),     # config 1 in full
    ([8, 8, 8, 8, 8], [4, 4, 4, 4], 10, 0.5),
    ([6] * 7, [5] * 6, 10, 0.0),             # config-4-like, 6^7
    ([16, 16, 16, 16], [8, 8, 8], 10, 1.0),
    ([7, 3, 11], [3, 5], 10, 0.0),
    # r > 8: step 2 (300 x 1200, r 12) takes the tensor-core path, steps 1 and 3 the generic one
    ([20, 30, 40, 30], [10, 12, 9], 10, 0.2),
    ([32, 16, 64, 8], [16, 24, 8], 6, 0.0),
]


@pytest.mark.parametrize("dims,ranks,iters,noise", NTT_CASES)
def test_decompose_parity(h, ora, dims, ranks, iters, noise):
    A = _tt_case(dims, ranks, 0, noise)
    ncore = ora.cores_size(dims, ranks)
    cores = torch.empty(ncore, dtype=torch.float32, device="cuda")
    e_dec = h.ntt_decompose(dev(A), dims, ranks, iters, 0, 1e-16, cores, want_error=True)
    got = host(cores)
    ref = ora.ntt_decompose(A, ranks, iters, seed=0)
    _cores_check(dims, ranks, got, ref)
    assert np.all(got >= 0)
    e_gpu = h.ntt_reconstruct(dims, ranks, cores, ref=dev(A), want_error=True)
    e_ora = ora.tt_rel_error(A, ranks, ref)
    assert abs(e_gpu - e_ora) <= 1e-3 * e_ora + 1e-6, (e_gpu, e_ora)
    assert abs(e_dec - e_gpu) <= 1e-9 + 1e-6 * e_gpu


def test_decompose_rank1_exact(h, ora):
    dims = [5, 4, 6, 3, 2]
    cores = (np.floor(ni.make_cores(dims, [1] * 4, seed=3) * 8) + 1) / 8
    A = ora.tt_full_f32(dims, [1] * 4, cores)
    out = torch.empty(ora.cores_size(dims, [1] * 4), dtype=torch.float32, device="cuda")
    h.ntt_decompose(dev(A), dims, [1] * 4, 1, 0, 1e-16, out)
    e = h.ntt_reconstruct(dims, [1] * 4, out, ref=dev(A), want_error=True)
    assert e < 1e-6


def test_decompose_host_pointers_and_workspace(h, ora):
    import paper_2008_01340_b200 as P
    dims, ranks = [6, 5, 4, 7], [3, 4, 2]
    A = _tt_case(dims, ranks, 1, 0.2)
    c_host = np.empty(ora.cores_size(dims, ranks), np.float32)
    h.ntt_decompose(A, dims, ranks, 10, 1, 1e-16, c_host)
    wsb = P.ntt_decompose_workspace_bytes(dims, ranks)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    c_dev = torch.empty_like(torch.from_numpy(c_host)).cuda()
    h.ntt_decompose(dev(A), dims, ranks, 10, 1, 1e-16, c_dev, ws, wsb)
    assert np.array_equal(host(c_dev), c_host)
    with pytest.raises(P.NttError) as e:
        h.ntt_decompose(dev(A), dims, ranks, 10, 1, 1e-16, c_dev, ws, wsb - 1)
    assert e.value.status == 6
    with pytest.raises(P.NttError) as e:
        h.ntt_decompose(dev(A), dims, [3, 40, 2], 10, 1, 1e-16, c_dev)
    assert e.value.status == 3


# ---------------------------------------------------- reconstruct / generate --
@pytest.mark.parametrize("dims,ranks", [([5, 4, 5, 6], [4, 3, 2]), ([3, 7], [2]), ([4] * 6, [3, 5, 2, 4, 3]),
                                        ([9, 1, 5, 2], [2, 2, 2]), ([3, 4], [2]), ([5, 8], [3]), ([7, 3, 16], [2, 3]),
                                        ([64, 64, 64], [5, 7])])
def test_reconstruct_parity(h, ora, dims, ranks):
    cores = ni.make_cores(dims, ranks, seed=2).astype(np.float32)
    out = torch.empty(int(np.prod(dims)), dtype=torch.float32, device="cuda")
    h.ntt_reconstruct(dims, ranks, dev(cores), out=out)
    ref = ora.tt_full(dims, ranks, cores.astype(np.float64)).ravel()
    got = host(out).astype(np.float64)
    assert np.all(np.abs(got - ref) <= 1e-5 * np.abs(ref).max())
    A = ora.tt_full_f32(dims, ranks, ni.make_cores(dims, ranks, seed=3), noise_amp=0.1, seed=3)
    e = h.ntt_reconstruct(dims, ranks, dev(cores), ref=dev(A), want_error=True)
    eo = ora.tt_rel_error(A, ranks, cores.astype(np.float64))
    assert abs(e - eo) <= 1e-5 * eo


@pytest.mark.parametrize("dims,ranks", [([32, 32, 32, 32], [3, 8, 5]),      # 16 items, 16 CTAs
                                        ([64, 64, 64, 64], [4, 16, 2]),     # 256 items on 148 CTAs
                                        ([16, 64, 64, 64], [2, 1, 7]),
                                        ([64, 64, 64, 64], [2, 12, 3])])
def test_error_stream_full_tiles(h, ora, dims, ranks):
    """Eq. 3 on split shapes with N_L % 64 == 0 and N_R % 1024 == 0: the error-only
    cp.async ring kernel (k_tt_err), incl. CTAs with several items and the zeroed spare partial
    slots (fewer CTAs than the plan's partials), against the oracle's fp64 error."""
    cores = ni.make_cores(dims, ranks, seed=7).astype(np.float32)
    A = ora.tt_full_f32(dims, ranks, ni.make_cores(dims, ranks, seed=8), noise_amp=0.2, seed=8)
    e = h.ntt_reconstruct(dims, ranks, dev(cores), ref=dev(A), want_error=True)
    eo = ora.tt_rel_error(A, ranks, cores.astype(np.float64))
    assert abs(e - eo) <= 1e-5 * eo
    e2 = h.ntt_reconstruct(dims, ranks, dev(cores), ref=dev(A), want_error=True)
    assert e2 == e  # fixed-order partial sums: bit-reproducible


def test_reconstruct_degenerate(h):
    import paper_2008_01340_b200 as P
    dims, ranks = [3, 4], [2]
    with pytest.raises(P.NttError) as e:
        h.ntt_reconstruct(dims, ranks, dev(np.ones(14, np.float32)), ref=dev(np.zeros(12, np.float32)), want_error=True)
    assert e.value.status == 4


def test_generate_matches_oracle_generator(h, ora):
    dims, ranks = [8, 6, 7, 5], [3, 4, 2]
    cores = ni.make_cores(dims, ranks, seed=5)
    out = torch.empty(int(np.prod(dims)), dtype=torch.float32, device="cuda")
    h.ntt_generate(dims, ranks, dev(cores.astype(np.float32)), 0.25, 5, 0x300, out)
    ref = ora.tt_full_f32(dims, ranks, cores, noise_amp=0.25, seed=5).ravel()
    assert np.allclose(host(out), ref, rtol=2e-6, atol=0)


@pytest.mark.parametrize("m,n,r", [(2, 4100, 2), (4, 60000, 4), (6, 70004, 5), (8, 1 << 16, 3), (1, 1024, 1),
                                   (6, 800, 6), (7, 4000, 4)])
def test_nmf_mu_small_path_parity(h, ora, m, n, r):
    """Very short unfoldings (m <= 8: config 4 step 1's shape class; k_fused with the 3-D X boxes,
    or direct H loads when n % 32 != 0) against the oracle."""
    X, W0, H0 = _mu_inputs(m, n, r, m * 11 + n)
    Xd, Wd, Hd = dev(X), dev(W0), dev(H0)
    h.ntt_nmf_mu(Xd, m, n, n, r, 10, 1e-16, Wd, Hd)
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), 10, eps=1e-16)
    assert_close_factor(host(Wd), Wo, what=f"small W {m}x{n} r{r}")
    assert_close_factor(host(Hd), Ho, what=f"small H {m}x{n} r{r}")


def test_validation_nonneg(h):
    """NTT_VALIDATE_NONNEG (SURVEY s.8(b)): with the flag on, a negative or NaN entry in
    X / A is rejected with NTT_ERR_NONNEG (status 5) before anything runs; valid input runs as
    without the flag (bit-identical); off by default."""
    import paper_2008_01340_b200 as P
    X, W0, H0 = _mu_inputs(8, 64, 2, 3)
    ref_W, ref_H = dev(W0), dev(H0)
    h.ntt_nmf_mu(dev(X), 8, 64, 64, 2, 3, 1e-16, ref_W, ref_H)
    h.ntt_set_validation(True)
    try:
        W, H = dev(W0), dev(H0)
        h.ntt_nmf_mu(dev(X), 8, 64, 64, 2, 3, 1e-16, W, H)
        assert torch.equal(W, ref_W) and torch.equal(H, ref_H)
        for bad in (-1e-3, float("nan")):
            Xb = X.copy()
            Xb[5, 17] = bad
            with pytest.raises(P.NttError) as e:
                h.ntt_nmf_mu(dev(Xb), 8, 64, 64, 2, 3, 1e-16, dev(W0), dev(H0))
            assert e.value.status == 5
            with pytest.raises(P.NttError) as e:
                h.ntt_nmf_bcd(dev(Xb), 8, 64, 64, 2, 3, dev(W0), dev(H0))
            assert e.value.status == 5
        dims, ranks = [5, 4, 5, 6], [4, 3, 2]
        A = _tt_case(dims, ranks)
        A.ravel()[123] = -0.5
        cores = torch.empty(P.cores_size(dims, ranks), device="cuda")
        for call in (lambda: h.ntt_decompose(dev(A), dims, ranks, 3, 0, 1e-16, cores),
                     lambda: h.ntt_decompose_bcd(dev(A), dims, ranks, 3, 0, cores)):
            with pytest.raises(P.NttError) as e:
                call()
            assert e.value.status == 5
    finally:
        h.ntt_set_validation(False)
    Xb = X.copy()
    Xb[0, 0] = -1.0
    h.ntt_nmf_mu(dev(Xb), 8, 64, 64, 2, 3, 1e-16, dev(W0), dev(H0))     # off: not checked


def test_nmf_mu_dynamic_tail(h, ora, monkeypatch):
    """k_fused_m's dynamic tail (the last ~64 tiles per CTA of every pass claimed at run time in
    groups of 16, each group's sums in a fixed slot): active from ~2.4 M columns on.  Bit-identical
    across runs (the claim order varies, the grouping does not), within rounding of the static
    schedule, and against the oracle at 1e-4."""
    m, n, r, iters = 32, 1 << 22, 8, 3
    assert h.mu_path(m, n, r) == 3
    X, W0, H0 = _mu_inputs(m, n, r, 4)
    Xd = dev(X)
    outs = []
    for tail in (True, True, False):
        if tail:
            monkeypatch.delenv("NTT_NO_TAIL", raising=False)
        else:
            monkeypatch.setenv("NTT_NO_TAIL", "1")
        Wd, Hd = dev(W0), dev(H0)
        h.ntt_nmf_mu(Xd, m, n, n, r, iters, 1e-16, Wd, Hd)
        outs.append((host(Wd), host(Hd)))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    for a, b in zip(outs[0], outs[2]):
        assert np.linalg.norm(a.astype(np.float64) - b) <= 1e-6 * np.linalg.norm(b)
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), iters, eps=1e-16)
    assert_close_factor(outs[0][0], Wo, what="W tail")
    assert_close_factor(outs[0][1], Ho, what="H tail")


def test_plan_paths_of_the_workloads(h):
    """Which kernel path plan_mu gives the TT steps of configs 3 and 4 and the paper's 256^4
    (ntt_debug_mu_path: 1 tiny, 2 cluster, 3 persistent one-pass); DESIGN.md s.6."""
    expect = {
        (32, 32 ** 5, 8): 3, (256, 32 ** 4, 8): 3, (256, 32 ** 3, 8): 3, (256, 32 ** 2, 8): 2, (256, 32, 8): 2,
        (6, 6 ** 9, 5): 3, (30, 6 ** 8, 5): 3, (30, 6 ** 7, 5): 3, (30, 6 ** 6, 5): 3, (30, 6 ** 5, 5): 3,
        (30, 6 ** 4, 5): 2, (30, 6 ** 3, 5): 2, (30, 36, 5): 1, (30, 6, 5): 1,
        (256, 256 ** 3, 10): 3,
    }
    got = {k: h.mu_path(*k) for k in expect}
    assert got == expect


def test_decompose_prefetch_input(h, ora):
    """ntt_prefetch_input: a host tensor staged into the next device slot on the copy stream is
    what a later ntt_decompose with that host pointer reads (two slots, oldest first), results
    bit-identical to the plain host-pointer call; a non-matching call copies its own input."""
    dims, ranks = [8, 8, 8, 8, 8], [4, 4, 4, 4]
    A1 = torch.from_numpy(_tt_case(dims, ranks, 1, 0.5)).pin_memory()
    A2 = torch.from_numpy(_tt_case(dims, ranks, 2, 0.5)).pin_memory()
    n = A1.numel()
    nc = ora.cores_size(dims, ranks)

    def run(A):
        c = torch.empty(nc, dtype=torch.float32).pin_memory()
        e = h.ntt_decompose(A, dims, ranks, 10, 0, 1e-16, c, want_error=True)
        return c.numpy().copy(), e

    r1, e1 = run(A1)
    r2, e2 = run(A2)
    h.ntt_prefetch_input(A1, n)
    h.ntt_prefetch_input(A2, n)
    g1, f1 = run(A1)
    g2, f2 = run(A2)
    assert np.array_equal(g1, r1) and np.array_equal(g2, r2) and f1 == e1 and f2 == e2
    h.ntt_prefetch_input(A1, n)
    g2b, _ = run(A2)   # no slot holds A2: the call copies it itself
    g1b, _ = run(A1)   # the slot staged above
    assert np.array_equal(g2b, r2) and np.array_equal(g1b, r1)
    import paper_2008_01340_b200 as P
    with pytest.raises(P.NttError):
        h.ntt_prefetch_input(torch.empty(4, device="cuda"), 4)
