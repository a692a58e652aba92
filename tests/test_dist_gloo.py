"""Multi-process (world_size 2, gloo, CPU) test of the distributed nTT scheme of
DESIGN.md s.7 -- the scheme libntt's NCCL path implements:

* the LAST tensor mode is block-partitioned (partition from libntt's host
  function ntt_dist_block), so every unfolding X_l is a column partition and the
  H -> X reshape stays local;
* H_l is initialised from the GLOBAL column index of each local column;
* each MU pass all-reduces the (X H^T, H H^T) partials; W is replicated;
* the last core is gathered from the ragged per-rank column blocks.

Each rank runs the scheme with the oracle's building blocks (fp64) and
torch.distributed.all_reduce / all_gather_object; the result must equal the
single-process oracle decomposition to rounding.
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


def global_cols(n_loc, b, nd, off):
    """Global column index of every local column of an unfolding whose last index is
    the last tensor mode, blocked as [off, off + b) (DESIGN.md s.7)."""
    c = np.arange(n_loc)
    return (c // b) * nd + off + (c % b)


def dist_ntt_scheme(A_local, dims, ranks, iters, seed, rank, world, off, b):
    import ntt_inputs as ni
    import oracle
    d = len(dims)
    fr = [1, *ranks, 1]
    T = A_local.astype(np.float64).ravel()
    cores = []
    rest_loc = T.size
    for l in range(1, d):
        m = fr[l - 1] * dims[l - 1]
        rest_loc //= dims[l - 1]
        n_loc = rest_loc
        n_glob = n_loc // b * dims[-1]
        r = fr[l]
        X = T.reshape(m, n_loc)
        W = ni.uniform(m * r, seed, ni.stream_w(l)).reshape(m, r)
        gc = global_cols(n_loc, b, dims[-1], off)
        H = np.empty((r, n_loc))
        for k in range(r):
            H[k] = ni.rng_u24(seed, ni.stream_h(l), (k * n_glob + gc).astype(np.uint64)) * 2.0 ** -24

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            dist.all_reduce(t)
            return t.numpy()

        for _ in range(iters):
            P = allreduce(oracle.xht(X, H))      # Alg. 5: local X H^T, summed over ranks
            Q = allreduce(oracle.gram_rows(H))   # Alg. 4
            W = oracle.w_update(W, P, Q)         # replicated W update
            G = oracle.gram_cols(W)              # W replicated: no communication
            S = oracle.wtx_cols(W, X)            # local columns only
            H = oracle.h_update_cols(H, S, G)
        cores.append(W.ravel())
        T = H.ravel()
    # last core: gather the ragged column blocks (Alg. 2 l.11)
    blocks = [None] * world
    dist.all_gather_object(blocks, (off, H))
    blocks.sort(key=lambda x: x[0])
    cores.append(np.concatenate([blk for _, blk in blocks], axis=1).ravel())
    return np.concatenate(cores)


def _worker(rank, world, port, dims, ranks, iters, outdir):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import ntt_inputs as ni
    import oracle
    import paper_2008_01340_b200 as P
    cores0 = ni.make_cores(dims, ranks, seed=3)
    A = oracle.tt_full_f32(dims, ranks, cores0, noise_amp=0.2, seed=3)
    b, off = P.ntt_dist_block(dims[-1], world, rank)   # libntt's partition
    A_local = np.ascontiguousarray(A[..., off:off + b])
    got = dist_ntt_scheme(A_local, dims, ranks, iters, seed=5, rank=rank, world=world, off=off, b=b)
    np.save(os.path.join(outdir, f"r{rank}.npy"), got)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("dims,ranks", [([4, 3, 5, 6], [3, 4, 2]), ([5, 4, 7], [3, 2]), ([3, 4, 3, 5], [2, 3, 3])])
def test_distributed_scheme_matches_serial_oracle(tmp_path, ora, dims, ranks):
    world, iters = 2, 6
    port = _free_port()
    mp.spawn(_worker, args=(world, port, dims, ranks, iters, str(tmp_path)), nprocs=world, join=True)
    import ntt_inputs as ni
    A = ora.tt_full_f32(dims, ranks, ni.make_cores(dims, ranks, seed=3), noise_amp=0.2, seed=3)
    ref = ora.ntt_decompose(A, ranks, iters, seed=5)
    outs = [np.load(tmp_path / f"r{g}.npy") for g in range(world)]
    assert np.array_equal(outs[0], outs[1])            # cores replicated on every rank
    assert np.allclose(outs[0], ref, rtol=1e-11, atol=1e-13)


def test_global_column_map_is_a_bijection():
    import paper_2008_01340_b200 as P
    dims = [4, 3, 7]
    for world in (1, 2, 3, 7):
        seen = []
        for g in range(world):
            b, off = P.ntt_dist_block(dims[-1], world, g)
            n_loc = dims[1] * b
            seen.append(global_cols(n_loc, b, dims[-1], off))
        allc = np.sort(np.concatenate(seen))
        assert np.array_equal(allc, np.arange(dims[1] * dims[2]))
