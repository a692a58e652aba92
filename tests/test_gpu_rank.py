"""GPU parity of the SVD rank rule (Alg. 2 l.5-6; SURVEY s.8(f) f2) and of
the eps-driven nTT sweep (ntt_decompose_eps) against the oracle.

The rank is an integer decided from floating point: inputs have clear spectral gaps
around every tested eps (reading R21), so the GPU (fp64 Gram eigenvalues) and the
oracle (LAPACK singular values) must pick the same rank exactly."""
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


def spectrum_matrix(s, m, n, seed=0):
    rng = np.random.default_rng(seed)
    U, _ = np.linalg.qr(rng.standard_normal((m, len(s))))
    V, _ = np.linalg.qr(rng.standard_normal((n, len(s))))
    return ((U * np.asarray(s, float)) @ V.T).astype(np.float32)


@pytest.mark.parametrize("m,n", [(6, 9), (9, 6), (40, 3000), (300, 700), (700, 200), (512, 4096)])
def test_rank_rule_known_spectrum(h, ora, m, n):
    N = min(m, n)
    s = np.concatenate([[10, 5, 1, 0.1, 0.01], 1e-4 * np.ones(N - 5)]) if N > 5 else np.array([10, 5, 1, 0.1, 0.01, 1e-3])[:N]
    X = spectrum_matrix(s, m, n)
    Xd = torch.from_numpy(X.ravel()).cuda()
    for eps in (2.0, 0.3, 0.05, 0.005, 3e-4):
        r_ora = ora.svd_tail_rank(X, eps)
        r_gpu, eig = h.ntt_rank_rule(Xd, m, n, n, eps, want_eig=True)
        assert r_gpu == r_ora, (m, n, eps, r_gpu, r_ora)
    sv = np.linalg.svd(X.astype(np.float64), compute_uv=False)
    ref = np.sort(sv ** 2)
    tot = ref.sum()
    assert np.abs(np.array(eig) - ref).max() <= 1e-12 * tot


@pytest.mark.parametrize("k", [1, 3, 8])
def test_rank_rule_exact_rank(h, ora, k):
    rng = np.random.default_rng(k)
    X = (rng.random((64, k)) @ rng.random((k, 5000))).astype(np.float32)
    r, _ = h.ntt_rank_rule(torch.from_numpy(X.ravel()).cuda(), 64, 5000, 5000, 1e-5)
    assert r == k == ora.svd_tail_rank(X, 1e-5)


def test_rank_rule_zero_and_large_eps(h):
    X = torch.zeros(10 * 20, device="cuda")
    assert h.ntt_rank_rule(X, 10, 20, 20, 0.1)[0] == 1
    Y = torch.rand(10 * 20, device="cuda")
    assert h.ntt_rank_rule(Y, 10, 20, 20, 1.5)[0] == 1


@pytest.mark.parametrize("dims,tranks,noise,eps_list", [
    ([5, 4, 5, 6], [4, 3, 2], 0.0, [0.5, 0.2, 0.05]),
    ([8, 6, 7, 5, 6], [3, 4, 4, 2], 0.0, [0.3, 0.1]),
    ([32, 32, 32], [6, 5], 0.02, [0.2, 0.05]),
])
def test_decompose_eps_parity(h, ora, dims, tranks, noise, eps_list):
    import paper_2008_01340_b200 as P
    A = ora.tt_full_f32(dims, tranks, ni.make_cores(dims, tranks, 1), noise_amp=noise, seed=1)
    Ad = torch.from_numpy(A.ravel()).cuda()
    cap = P.cores_size(dims, [64] * (len(dims) - 1))
    for tt_eps in eps_list:
        cores = torch.zeros(cap, device="cuda")
        ranks, err = h.ntt_decompose_eps(Ad, dims, tt_eps, 10, 3, 1e-16, cores, cap, want_error=True)
        r_ora, c_ora = ora.ntt_decompose_eps(A, tt_eps, iters=10, seed=3)
        assert ranks == r_ora, (tt_eps, ranks, r_ora)
        got = cores.cpu().numpy()[: c_ora.size].astype(np.float64)
        fro = np.linalg.norm(got - c_ora) / np.linalg.norm(c_ora)
        assert fro <= 1e-4, (tt_eps, fro)
        e_ora = ora.tt_rel_error(A, r_ora, c_ora)
        assert abs(err - e_ora) <= 1e-3 * e_ora + 1e-6
        # the fixed-rank path with the chosen ranks gives the same cores
        c2 = torch.empty(P.cores_size(dims, ranks), device="cuda")
        h.ntt_decompose(Ad, dims, ranks, 10, 3, 1e-16, c2)
        assert np.array_equal(c2.cpu().numpy(), cores.cpu().numpy()[: c2.numel()])


def test_decompose_eps_max_ranks_and_capacity(h):
    import paper_2008_01340_b200 as P
    dims = [6, 5, 7, 4]
    A = torch.rand(int(np.prod(dims)), device="cuda")
    cores = torch.zeros(P.cores_size(dims, [64] * 3), device="cuda")
    ranks, _ = h.ntt_decompose_eps(A, dims, 1e-6, 3, 0, 1e-16, cores, cores.numel(), max_ranks=[2, 3, 2])
    assert ranks[0] <= 2 and ranks[1] <= 3 and ranks[2] <= 2
    with pytest.raises(P.NttError):
        h.ntt_decompose_eps(A, dims, 1e-6, 3, 0, 1e-16, cores, 3)


# ---- min(m, n) > 512: the grid-wide Householder reduction + warp multisection (tt_rank.cu) ----
@pytest.mark.parametrize("m,n", [(600, 2000), (2000, 700), (1500, 1600), (2560, 2600)])
def test_rank_rule_grid_known_spectrum(h, ora, m, n):
    N = min(m, n)
    s = np.concatenate([[10, 5, 1, 0.1, 0.01], 1e-4 * np.ones(N - 5)])
    X = spectrum_matrix(s, m, n, seed=m + n)
    Xd = torch.from_numpy(X.ravel()).cuda()
    for eps in (2.0, 0.3, 0.05, 0.005, 3e-4):
        r_ora = ora.svd_tail_rank(X, eps)
        r_gpu, eig = h.ntt_rank_rule(Xd, m, n, n, eps, want_eig=True)
        assert r_gpu == r_ora, (m, n, eps, r_gpu, r_ora)
    sv = np.linalg.svd(X.astype(np.float64), compute_uv=False)
    ref = np.sort(sv ** 2)
    assert np.abs(np.array(eig) - ref).max() <= 1e-12 * ref.sum()


def test_rank_rule_grid_graded_spectrum(h, ora):
    """A geometric spectrum (no flat tail): every eps picks a different rank, and the
    eigenvalues match LAPACK's squared singular values to 1e-12 of the trace."""
    m, n = 900, 1200
    s = 0.7 ** np.arange(m)
    X = spectrum_matrix(s, m, n, seed=5)
    Xd = torch.from_numpy(X.ravel()).cuda()
    for eps in (0.5, 0.2, 0.1, 0.03, 0.01, 3e-3):
        assert h.ntt_rank_rule(Xd, m, n, n, eps)[0] == ora.svd_tail_rank(X, eps)


def test_decompose_eps_grid_step(h, ora):
    """ntt_decompose_eps with a first unfolding of 600 x 1000 (grid path) on a non-negative
    exact rank-4 tensor: ranks identical to the oracle's, cores within 1e-4."""
    import paper_2008_01340_b200 as P
    dims = [600, 10, 100]
    rng = np.random.default_rng(11)
    A = (rng.random((600, 4)) @ rng.random((4, 1000))).astype(np.float32).reshape(dims)
    Ad = torch.from_numpy(A.ravel()).cuda()
    cap = P.cores_size(dims, [64] * 2)
    for tt_eps in (0.3, 1e-4):
        cores = torch.zeros(cap, device="cuda")
        ranks, err = h.ntt_decompose_eps(Ad, dims, tt_eps, 10, 3, 1e-16, cores, cap, want_error=True)
        r_ora, c_ora = ora.ntt_decompose_eps(A, tt_eps, iters=10, seed=3)
        assert ranks == r_ora, (tt_eps, ranks, r_ora)
        got = cores.cpu().numpy()[: c_ora.size].astype(np.float64)
        assert np.linalg.norm(got - c_ora) / np.linalg.norm(c_ora) <= 1e-4
        e_ora = ora.tt_rel_error(A, r_ora, c_ora)
        assert abs(err - e_ora) <= 1e-3 * e_ora + 1e-6


def test_rank_rule_limit(h):
    import paper_2008_01340_b200 as P
    X = torch.zeros(4097 * 4100, device="cuda")
    with pytest.raises(P.NttError):
        h.ntt_rank_rule(X, 4097, 4100, 4100, 0.1)
