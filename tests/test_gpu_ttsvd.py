"""GPU parity of the TT-SVD baseline (SURVEY s.8(f) f4; reading R28)
against oracle.tt_svd.

Singular vectors are unique up to sign when the singular values at and above each cut are
distinct; both sides fix the sign the same way (largest-|entry| of a core column positive),
so cores compare element by element.  Ranks are integers decided from floating point: the
inputs keep clear spectral gaps around the chosen eps (as for the rank rule, R21).
Tolerances: cores and reconstruction 1e-4 relative to their max entry (fp32 storage,
fp64 Gram and eigensolver); ranks exact; Eq. 3 error within 1e-3 relative (R15)."""
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


def rand_tt(dims, ranks, seed, noise=0.0):
    rng = np.random.default_rng(seed)
    rr = [1] + list(ranks) + [1]
    out = None
    for l, n in enumerate(dims):
        G = rng.standard_normal((rr[l], n, rr[l + 1]))
        out = G.reshape(n, -1) if out is None else (out.reshape(-1, rr[l]) @ G.reshape(rr[l], -1))
    A = out.reshape(dims)
    if noise:
        A = A + noise * np.abs(A).mean() * rng.standard_normal(dims)
    return A.astype(np.float32)


def run(h, A, eps, max_ranks=None):
    import paper_2008_01340_b200 as P
    dims = list(A.shape)
    cap = P.cores_size(dims, [64] * (len(dims) - 1))
    cores = torch.empty(cap, device="cuda")
    ranks, err = h.ntt_tt_svd(torch.from_numpy(A.ravel()).cuda(), dims, eps, cores, cap, max_ranks=max_ranks,
                              want_error=True)
    return ranks, cores[: P.cores_size(dims, ranks)].cpu().numpy(), err


def compare(ora, A, eps, ranks, cores, err, max_ranks=None):
    dims = list(A.shape)
    ro, co, tails = ora.tt_svd(A.astype(np.float64), eps, max_ranks)
    assert list(ranks) == list(ro)
    assert np.abs(cores - co).max() <= 1e-4 * np.abs(co).max()
    B = ora.tt_full(dims, ranks, cores.astype(np.float64))
    Bo = ora.tt_full(dims, ro, co)
    assert np.abs(B - Bo).max() <= 1e-4 * np.abs(Bo).max()
    e_ora = ora.rel_error(A, Bo)
    assert abs(err - e_ora) <= 1e-3 * e_ora + 1e-6
    return ro, tails


@pytest.mark.parametrize("dims,tr,noise,eps", [
    ((6, 5, 7, 4), (3, 4, 2), 0.01, 0.05),
    ((4, 4, 4, 4, 4), (3, 5, 5, 3), 0.02, 0.1),
    ((8, 8, 3), (5, 3), 0.01, 0.05),          # last step m = 40 > n = 3: the X V / s branch
    ((3, 40, 50), (3, 6), 0.0, 1e-4),
    ((12, 10, 9, 8), (6, 9, 5), 0.005, 0.02)])
def test_ttsvd_parity(h, ora, dims, tr, noise, eps):
    A = rand_tt(dims, tr, sum(dims), noise)
    ranks, cores, err = run(h, A, eps)
    compare(ora, A, eps, ranks, cores, err)
    assert list(ranks) == list(tr)            # the gaps put the cut at the true ranks


def test_ttsvd_caps_and_full_rank(h, ora):
    A = rand_tt((6, 7, 5), (4, 4), 3, 0.05)
    ranks, cores, err = run(h, A, 0.0, max_ranks=[3, 2])
    assert ranks == [3, 2]
    compare(ora, A, 0.0, ranks, cores, err, max_ranks=[3, 2])
    ranks, cores, err = run(h, A, 0.0)        # full ranks: exact up to fp32
    assert ranks == [6, 5]
    assert err <= 1e-5


def test_ttsvd_larger_and_error_decomposition(h, ora):
    """16^5 tensor of TT ranks 6 + noise (several Gram tiles, split-K passes, ragged
    column blocks): parity with the oracle, and the error equals the root of the summed
    per-step discarded energies (the orthogonality of the left cores)."""
    dims = [16] * 5
    A = rand_tt(dims, (6, 6, 6, 6), 11, 0.01)
    ranks, cores, err = run(h, A, 0.01)
    ro, tails = compare(ora, A, 0.01, ranks, cores, err)
    nA2 = float(np.sum(A.astype(np.float64) ** 2))
    assert abs(err - np.sqrt(tails.sum() / nA2)) <= 1e-3 * err + 1e-6


def test_ttsvd_unsupported(h):
    """min(m, n) above the eigensolver's 4096 limit is rejected."""
    import paper_2008_01340_b200 as P
    A = torch.zeros(4100 * 4100, device="cuda")
    cores = torch.empty(10 ** 6, device="cuda")
    with pytest.raises(P.NttError):
        h.ntt_tt_svd(A, [4100, 4100], 0.1, cores, 10 ** 6)


def test_ttsvd_host_buffers(h, ora):
    """Host A and host cores (staged by the library) give the same result as device buffers."""
    import paper_2008_01340_b200 as P
    A = rand_tt((6, 5, 7, 4), (3, 4, 2), 5, 0.01)
    dims = list(A.shape)
    cap = P.cores_size(dims, [64] * 3)
    cd = torch.empty(cap, device="cuda")
    rd, ed = h.ntt_tt_svd(torch.from_numpy(A.ravel()).cuda(), dims, 0.05, cd, cap, want_error=True)
    ch = np.empty(cap, dtype=np.float32)
    rh, eh = h.ntt_tt_svd(np.ascontiguousarray(A.ravel()), dims, 0.05, ch, cap, want_error=True)
    k = P.cores_size(dims, rd)
    assert rd == rh and ed == eh and np.array_equal(cd.cpu().numpy()[:k], ch[:k])


def test_ttsvd_large_ranks(h, ora):
    """Ranks above 32 (the 64-rank classes of the X' = U^T X kernel and the eigensolver's
    64-vector Rayleigh-Ritz) on an exact TT of ranks (40, 30) + small noise."""
    A = rand_tt((48, 50, 40), (40, 30), 21, 1e-3)
    ranks, cores, err = run(h, A, 1e-3)
    compare(ora, A, 1e-3, ranks, cores, err)
    assert ranks == [40, 30]


@pytest.mark.parametrize("dims,tr,noise,eps", [
    ((600, 10, 100), (5, 4), 0.001, 0.01),     # step 1: 600 x 1000 (grid-wide eigensolver)
    ((40, 30, 1200), (20, 12), 0.001, 0.01),   # step 2: 600 x 1200 (m = r1 n2 = 600 > 512)
    ((1100, 2, 1000), (6, 3), 0.0005, 0.01)])  # step 1: 1100 x 2000
def test_ttsvd_parity_grid_eigensolver(h, ora, dims, tr, noise, eps):
    """min(m, n) > 512 at a step: the grid-wide Householder reduction (reflectors kept), the warp
    multisection, k_svd_vec (inverse iteration, CGS2, Rayleigh-Ritz) and k_backtransform --
    ranks identical to LAPACK's, cores, reconstruction and Eq. 3 as the one-CTA path."""
    A = rand_tt(dims, tr, sum(dims), noise)
    ranks, cores, err = run(h, A, eps)
    compare(ora, A, eps, ranks, cores, err)
    assert list(ranks) == list(tr)
