"""TT-SVD baseline (ntt_tt_svd, SURVEY s.8(f) f4) timing on BASELINE configs 3 and 4
next to the nTT sweep at the same ranks (tools only).

    python tools/bench_ttsvd.py [config3|config4] [reps]
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

which = sys.argv[1:2] or ["config3", "config4"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
h = P.Handle(0)
for name in which:
    w = ni.workloads()[name]
    cores0 = torch.from_numpy(ni.make_cores(w.dims, w.ranks, w.seed).astype(np.float32)).cuda()
    A = torch.empty(w.numel, device="cuda")
    h.ntt_generate(w.dims, w.ranks, cores0, w.noise_amp, w.seed, ni.STREAM_NOISE, A)
    cap = P.cores_size(w.dims, [64] * (len(w.dims) - 1))
    cores = torch.empty(cap, device="cuda")
    ranks, err = h.ntt_tt_svd(A, w.dims, 0.0, cores, cap, max_ranks=w.ranks, want_error=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        h.ntt_tt_svd(A, w.dims, 0.0, cores, cap, max_ranks=w.ranks)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    nc = torch.empty(P.cores_size(w.dims, w.ranks), device="cuda")
    err_ntt = h.ntt_decompose(A, w.dims, w.ranks, w.iters, w.seed, 1e-16, nc, want_error=True)
    print(json.dumps({"workload": name, "dims": w.dims, "ranks": ranks, "ttsvd_ms": ms, "ttsvd_rel_err": err,
                      "ntt_mu_rel_err": err_ntt, "A_GB": 4.0 * w.numel / 1e9}), flush=True)
    del A, cores, nc
    torch.cuda.empty_cache()
