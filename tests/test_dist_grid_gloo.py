"""Multi-process (gloo, CPU) test of the 2-D pr x pc NMF grid of DESIGN.md s.7 /
SURVEY s.8(e) -- the scheme libntt's NCCL path (ntt_create_dist_grid +
ntt_nmf_mu) implements for the plain NMF (BASELINE config 5):

* rank = ga * pc + gb holds X[rows of block ga, cols of block gb] (blocks from
  libntt's ntt_dist_block), W rows of block ga, H columns of block gb;
* per iteration: all-reduce of (X H^T, H H^T) over the grid row, of W^T W and of
  the W^T X block over the grid column (Alg. 5 / Alg. 6 / Alg. 4 with the
  reduce-scatter + all-gather pairs written as all-reduces); X never moves.

Each rank runs the scheme with the oracle's building blocks (fp64); the gathered
factors must equal the single-process oracle NMF to rounding.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def inputs(m, n, r, seed=4):
    import ntt_inputs as ni
    rng = np.random.default_rng(seed)
    X = (rng.random((m, r)) @ rng.random((r, n)) + 0.05 * rng.random((m, n))).astype(np.float32)
    W0 = ni.uniform(m * r, seed, ni.stream_w(1)).reshape(m, r)
    H0 = ni.uniform(r * n, seed, ni.stream_h(1)).reshape(r, n)
    return X, W0, H0


def grid_scheme(X, W0, H0, iters, pr, pc, ga, gb, row_group, col_group):
    import oracle
    import paper_2008_01340_b200 as P
    m, n = X.shape
    bm, om = P.ntt_dist_block(m, pr, ga)
    bn, on = P.ntt_dist_block(n, pc, gb)
    Xl = X[om:om + bm, on:on + bn].astype(np.float64)
    W = W0[om:om + bm].copy()
    H = H0[:, on:on + bn].copy()

    def allreduce(a, group):
        t = torch.from_numpy(np.ascontiguousarray(a))
        dist.all_reduce(t, group=group)
        return t.numpy()

    for _ in range(iters):
        PQ = allreduce(np.concatenate([oracle.xht(Xl, H).ravel(), oracle.gram_rows(H).ravel()]), row_group)
        r = W.shape[1]
        Pm, Q = PQ[:bm * r].reshape(bm, r), PQ[bm * r:].reshape(r, r)
        W = oracle.w_update(W, Pm, Q)
        G = allreduce(oracle.gram_cols(W), col_group)
        S = allreduce(oracle.wtx_cols(W, Xl), col_group)
        H = oracle.h_update_cols(H, S, G)
    return (om, W), (on, H)


def _worker(rank, world, port, pr, pc, shape, iters, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ga, gb = rank // pc, rank % pc
    rows = [dist.new_group([a * pc + b for b in range(pc)]) for a in range(pr)]
    cols = [dist.new_group([a * pc + b for a in range(pr)]) for b in range(pc)]
    m, n, r = shape
    X, W0, H0 = inputs(m, n, r)
    (om, W), (on, H) = grid_scheme(X, W0, H0, iters, pr, pc, ga, gb, rows[ga], cols[gb])
    np.save(os.path.join(outdir, f"W{rank}.npy"), W)
    np.save(os.path.join(outdir, f"H{rank}.npy"), H)
    with open(os.path.join(outdir, f"off{rank}.txt"), "w") as f:
        f.write(f"{om} {on}")
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("pr,pc,shape", [(2, 1, (13, 9, 3)), (1, 2, (7, 15, 2)), (2, 2, (11, 10, 3))])
def test_grid_nmf_scheme_matches_serial_oracle(tmp_path, ora, pr, pc, shape):
    world, iters = pr * pc, 7
    mp.spawn(_worker, args=(world, _free_port(), pr, pc, shape, iters, str(tmp_path)), nprocs=world, join=True)
    m, n, r = shape
    X, W0, H0 = inputs(m, n, r)
    Wo, Ho = ora.nmf_mu(X, W0, H0, iters)
    W = np.zeros_like(Wo)
    H = np.zeros_like(Ho)
    for g in range(world):
        om, on = map(int, open(tmp_path / f"off{g}.txt").read().split())
        Wl, Hl = np.load(tmp_path / f"W{g}.npy"), np.load(tmp_path / f"H{g}.npy")
        # replicated blocks agree across their group to rounding
        if np.any(W[om:om + Wl.shape[0]]):
            assert np.allclose(W[om:om + Wl.shape[0]], Wl, rtol=1e-13, atol=0)
        if np.any(H[:, on:on + Hl.shape[1]]):
            assert np.allclose(H[:, on:on + Hl.shape[1]], Hl, rtol=1e-13, atol=0)
        W[om:om + Wl.shape[0]] = Wl
        H[:, on:on + Hl.shape[1]] = Hl
    assert np.allclose(W, Wo, rtol=1e-11, atol=1e-13)
    assert np.allclose(H, Ho, rtol=1e-11, atol=1e-13)
