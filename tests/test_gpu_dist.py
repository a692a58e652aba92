"""The library's distributed path (ntt_create_dist / ntt_create_dist_grid) on one GPU.

A handle made by ntt_create_dist* always takes the distributed branches, also with
a 1-rank communicator.  The per-pass cross-GPU reduction of the fp64 (X H^T, H H^T)
partials runs either inside the persistent kernels (ntt_set_dist_exchange mode 1,
the default: NVLink peer stores into the ranks' IPC-mapped exchange buffers, release /
acquire flags, rank-order sum; ntt_peer_exchange_count proves the device did it) or
as a per-pass ncclAllReduce between kernel launches (mode 0, dist_reduce); then the
global-column-index H init
(k_fill_uniform_cols), the last-core gather by per-rank broadcasts into a staging
area plus k_gather_last_core, the all-reduce of the Eq. 3 sums, and on the
tensor-core path tc_reduce_PQ / tc_wupdate_ex / tc_reduce_S / tc_hupdate_ex over
the grid-row and grid-column communicators.  ntt_collective_count proves the NCCL
calls were issued.  Results must match the single-GPU handle and the oracle (parity
tolerances of test_gpu_parity).  The p > 1 index maps of the init and of the gather
are checked at kernel level on emulated layouts (p = 8, rank 3; ragged n_d = 7 over
p = 3)."""
import numpy as np
import pytest

import ntt_inputs as ni

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def handles():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2008_01340_b200 as P
    uid = P.ntt_get_unique_id()
    hd = P.Handle(0, unique_id=uid, nranks=1, rank=0)
    assert hd.size == 1 and hd.rank == 0
    return P.Handle(0), hd


@pytest.mark.parametrize("dims,ranks,iters", [([5, 4, 5, 6], [4, 3, 2], 10), ([16, 16, 16, 16], [8, 8, 8], 10),
                                              ([6] * 6, [5] * 5, 10), ([64, 32, 64], [8, 8], 5),
                                              ([20, 30, 40, 30], [10, 12, 9], 5)])
@pytest.mark.parametrize("mode", [0, 1])
def test_dist_handle_decompose_matches(handles, ora, dims, ranks, iters, mode):
    h1, hd = handles
    hd.ntt_set_dist_exchange(mode)
    A = ora.tt_full_f32(dims, ranks, ni.make_cores(dims, ranks, 0), noise_amp=0.3, seed=0)
    Ad = torch.from_numpy(A).cuda()
    c1 = torch.empty(ora.cores_size(dims, ranks), device="cuda")
    cd = torch.empty_like(c1)
    e1 = h1.ntt_decompose(Ad, dims, ranks, iters, 0, 1e-16, c1, want_error=True)
    n0, x0 = hd.collective_count, hd.peer_exchange_count
    ed = hd.ntt_decompose(Ad, dims, ranks, iters, 0, 1e-16, cd, want_error=True)
    if mode == 0:
        # per MU pass one all-reduce; a graph replay of an identical call issues none anew
        assert hd.collective_count - n0 >= (len(dims) - 1) * iters
    else:
        # steps on a persistent one-pass kernel exchange inside it (one per pass), the others
        # (n % 4 != 0, tall / square unfoldings) all-reduce per pass
        nx = hd.peer_exchange_count - x0
        assert nx % iters == 0
        if dims == [16, 16, 16, 16]:  # m = 16 and 128 at r = 8: all three steps persistent
            assert nx == 3 * iters
        assert nx + (hd.collective_count - n0) >= (len(dims) - 1) * iters
    torch.cuda.synchronize()
    a, b = c1.cpu().numpy().astype(np.float64), cd.cpu().numpy().astype(np.float64)
    assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(a)
    ref = ora.ntt_decompose(A, ranks, iters, seed=0)
    assert np.linalg.norm(b - ref) <= 1e-4 * np.linalg.norm(ref)
    assert abs(ed - e1) <= 1e-5 * e1
    hd.ntt_set_dist_exchange(1)


@pytest.mark.parametrize("m,n,r", [(32, 4096, 8), (256, 2048, 8), (100, 700, 16), (8, 4096, 4), (40, 1024, 8),
                                   (256, 4096, 12), (64, 2048, 8),
                                   (32, 1 << 22, 8)])  # k_fused_m with its dynamic tail + the exchange
@pytest.mark.parametrize("mode", [0, 1])
def test_dist_handle_nmf_mu(handles, ora, m, n, r, mode, monkeypatch):
    h1, hd = handles
    hd.ntt_set_dist_exchange(mode)
    rng = np.random.default_rng(1)
    X = rng.random((m, n)).astype(np.float32)
    W0 = ni.uniform(m * r, 1, 0x202).reshape(m, r).astype(np.float32)
    H0 = ni.uniform(r * n, 1, 0x203).reshape(r, n).astype(np.float32)
    Xd = torch.from_numpy(X).cuda()
    Wd, Hd = torch.from_numpy(W0.copy()).cuda(), torch.from_numpy(H0.copy()).cuda()
    n0, x0 = hd.collective_count, hd.peer_exchange_count
    hd.ntt_nmf_mu(Xd, m, n, n, r, 8, 1e-16, Wd, Hd)
    if mode == 0:  # every shape here runs a persistent one-pass kernel on mode 1
        assert hd.collective_count - n0 >= 8
    else:
        assert hd.collective_count == n0 and hd.peer_exchange_count - x0 == 8
        # 1 rank: the rank-order sum of one vector is that vector, so the in-kernel exchange is
        # bit-identical to the single-GPU persistent kernel (cluster mode, which single-GPU
        # handles take for some of these shapes, sums in another order)
        monkeypatch.setenv("NTT_NO_CLUSTER", "1")
        W1, H1 = torch.from_numpy(W0.copy()).cuda(), torch.from_numpy(H0.copy()).cuda()
        h1.ntt_nmf_mu(Xd, m, n, n, r, 8, 1e-16, W1, H1)
        assert torch.equal(W1, Wd) and torch.equal(H1, Hd)
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), 8)
    W, H = Wd.cpu().numpy(), Hd.cpu().numpy()
    assert np.linalg.norm(W - Wo) <= 1e-4 * np.linalg.norm(Wo)
    assert np.linalg.norm(H - Ho) <= 1e-4 * np.linalg.norm(Ho)
    hd.ntt_set_dist_exchange(1)


@pytest.mark.parametrize("m,n,r", [(512, 1024, 16), (1000, 776, 32)])
def test_grid_handle_tc_nmf_matches(handles, ora, m, n, r):
    """2-D grid handle (1 x 1 on one GPU): the tensor-core NMF path with the grid-row /
    grid-column NCCL all-reduces must be bit-identical to the single-GPU path (the
    split partials are summed in the same order) and match the oracle."""
    import paper_2008_01340_b200 as P
    h1, _ = handles
    hg = P.Handle(0, unique_id=P.ntt_get_unique_id(), nranks=1, rank=0, grid=(1, 1))
    assert hg.grid == (1, 1, 0, 0)
    rng = np.random.default_rng(2)
    X = (rng.random((m, r)) @ rng.random((r, n)) + 0.01 * rng.random((m, n))).astype(np.float32)
    W0 = ni.uniform(m * r, 2, 0x202).reshape(m, r).astype(np.float32)
    H0 = ni.uniform(r * n, 2, 0x203).reshape(r, n).astype(np.float32)
    Xd = torch.from_numpy(X).cuda()
    outs = []
    for h in (h1, hg):
        Wd, Hd = torch.from_numpy(W0.copy()).cuda(), torch.from_numpy(H0.copy()).cuda()
        h.ntt_profile_enable(True)
        n0 = h.collective_count
        h.ntt_nmf_mu(Xd, m, n, n, r, 6, 1e-16, Wd, Hd)
        # grid handle: 3 all-reduces per iteration (row: X H^T | H H^T; column: W^T W, W^T X)
        assert h.collective_count - n0 == (18 if h is hg else 0)
        assert h.ntt_profile_get(6)[0] == 6, "tensor-core path not taken"
        h.ntt_profile_enable(False)
        outs.append((Wd.cpu().numpy(), Hd.cpu().numpy()))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), 6)
    assert np.linalg.norm(outs[1][0] - Wo) <= 1e-4 * np.linalg.norm(Wo)
    assert np.linalg.norm(outs[1][1] - Ho) <= 1e-4 * np.linalg.norm(Ho)


def test_grid_handle_rejects_bad_grid():
    import paper_2008_01340_b200 as P
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    with pytest.raises(P.NttError):
        P.Handle(0, unique_id=P.ntt_get_unique_id(), nranks=1, rank=0, grid=(2, 1))


@pytest.mark.parametrize("dims,ranks,p,g", [([5, 4, 6, 16], [3, 4, 2], 8, 3), ([4, 3, 7], [2, 3], 3, 2),
                                            ([4, 3, 7], [2, 3], 3, 0), ([6, 5, 9], [4, 2], 4, 1)])
def test_fill_uniform_cols_layout(handles, dims, ranks, p, g):
    """k_fill_uniform_cols on the local H of rank g of p (last mode block-partitioned,
    DESIGN.md s.7): every entry equals the RNG spec drawn at the GLOBAL index of
    ntt_inputs.rng_u24, at every TT step, so inits agree for any p."""
    import paper_2008_01340_b200 as P
    _, hd = handles
    nd = dims[-1]
    b, off = P.ntt_dist_block(nd, p, g)
    rest = int(np.prod(dims))
    for l in range(1, len(dims)):
        rest //= dims[l - 1]
        r = ranks[l - 1]
        nglob = rest
        nloc = rest // nd * b
        H = torch.empty(r * nloc, device="cuda")
        hd.ntt_debug_fill_uniform_cols(H, r, nloc, b, nd, off, nglob, 7, ni.stream_h(l))
        c = np.arange(nloc)
        cg = (c // b) * nd + off + c % b
        idx = (np.arange(r)[:, None] * nglob + cg[None, :]).ravel()
        ref = ni.rng_u24(7, ni.stream_h(l), idx).astype(np.float64) * 2.0 ** -24
        assert np.array_equal(H.cpu().numpy().astype(np.float64), ref)


@pytest.mark.parametrize("r,nd,p", [(3, 7, 3), (2, 16, 8), (5, 9, 4), (1, 5, 5)])
def test_gather_last_core_ragged(handles, r, nd, p):
    """k_gather_last_core: rank-major staging [rank g: r x b_g] -> core[k][i] (r x nd) for
    ragged blocks b_g = floor((g+1) nd / p) - floor(g nd / p)."""
    import paper_2008_01340_b200 as P
    _, hd = handles
    core = np.arange(r * nd, dtype=np.float32).reshape(r, nd) + 1
    blocks = [P.ntt_dist_block(nd, p, g) for g in range(p)]
    assert sum(b for b, _ in blocks) == nd
    gath = np.concatenate([core[:, o:o + b].ravel() for b, o in blocks])
    out = torch.full((r * nd,), -1.0, device="cuda")
    hd.ntt_debug_gather_last_core(torch.from_numpy(gath).cuda(), r, nd, p, out)
    assert np.array_equal(out.cpu().numpy().reshape(r, nd), core)


def test_dist_handle_generic_split_k(handles, ora):
    """The generic two-pass path with the split-K H pass on a 1-rank NCCL handle (per-pass
    all-reduce of the (X H^T, H H^T) vector, then the W update and the split H pass; the split
    pass reuses the reduced vector's buffer for G): oracle parity and agreement with the
    single-GPU handle."""
    h1, hd = handles
    m, n, r, it = 3000, 200, 20, 8
    rng = np.random.default_rng(3)
    X = rng.random((m, n)).astype(np.float32)
    W0 = ni.uniform(m * r, 3, 0x202).reshape(m, r).astype(np.float32)
    H0 = ni.uniform(r * n, 3, 0x203).reshape(r, n).astype(np.float32)
    Xd = torch.from_numpy(X).cuda()
    outs = []
    for h in (h1, hd):
        Wd, Hd = torch.from_numpy(W0.copy()).cuda(), torch.from_numpy(H0.copy()).cuda()
        n0 = h.collective_count
        h.ntt_nmf_mu(Xd, m, n, n, r, it, 1e-16, Wd, Hd)
        if h is hd:
            assert h.collective_count - n0 >= it
        outs.append((Wd.cpu().numpy(), Hd.cpu().numpy()))
    Wo, Ho = ora.nmf_mu(X, W0.astype(np.float64), H0.astype(np.float64), it)
    for W, H in outs:
        assert np.linalg.norm(W - Wo) <= 1e-4 * np.linalg.norm(Wo)
        assert np.linalg.norm(H - Ho) <= 1e-4 * np.linalg.norm(Ho)
    assert np.linalg.norm(outs[0][1] - outs[1][1]) <= 1e-5 * np.linalg.norm(outs[0][1])
