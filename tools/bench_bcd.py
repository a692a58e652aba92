"""BCD NMF (Alg. 3, ntt_nmf_bcd) timing next to MU on BASELINE configs 2 and 5 (tools only).

    python tools/bench_bcd.py [config2|config5] [iters]

Config 5 at 1 GPU runs on the 32768 x 65536 row slice.  X = W0 H0 + noise from ntt_generate.
Algorithmic bytes per BCD iteration: two reads of X (W^T X in the H step, X H^T for the
objective / next W step) = 8 m n, plus O((m + n) r) factor traffic.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

which = sys.argv[1:2] or ["config2", "config5"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
h = P.Handle(0)
for name in which:
    w = ni.workloads()[name]
    m, n = w.dims
    r = min(w.ranks[0], 32)
    if name == "config5":
        m = 32768
    dims, ranks, cores = ni.make_factor_cores(m, n, r, 0)
    X = torch.empty(m * n, device="cuda")
    h.ntt_generate(dims, ranks, torch.from_numpy(cores.astype(np.float32)).cuda(), w.noise_amp or 0.01, 0,
                   ni.STREAM_NOISE, X)
    W0 = torch.empty(m * r, device="cuda")
    H0 = torch.empty(r * n, device="cuda")
    h.ntt_fill_uniform(W0, m * r, 0, ni.stream_w(1))
    h.ntt_fill_uniform(H0, r * n, 0, ni.stream_h(1))
    row = {"workload": name, "m": m, "n": n, "r": r, "iters": iters}
    for _ in range(2):  # warm both paths (clocks, graph capture, workspace) before timing either
        W, H = W0.clone(), H0.clone()
        h.ntt_nmf_bcd(X, m, n, n, r, iters, W, H)
        h.ntt_nmf_mu(X, m, n, n, r, iters, 1e-16, W, H)
    torch.cuda.synchronize()
    for alg in ("bcd", "mu"):
        W, H = W0.clone(), H0.clone()
        if alg == "bcd":
            h.ntt_nmf_bcd(X, m, n, n, r, 2, W, H)
        else:
            h.ntt_nmf_mu(X, m, n, n, r, 2, 1e-16, W, H)
        W, H = W0.clone(), H0.clone()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        if alg == "bcd":
            tr = h.ntt_nmf_bcd(X, m, n, n, r, iters, W, H, trace=True)
        else:
            h.ntt_nmf_mu(X, m, n, n, r, iters, 1e-16, W, H)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        Xm = X.view(m, n)
        err = float(torch.linalg.norm(Xm - W.view(m, r) @ H.view(r, n)) / torch.linalg.norm(Xm))
        row[alg] = {"ms_per_iter": ms, "it_per_s": 1e3 / ms, "rel_err": err,
                    "GBps_2xX": 8.0 * m * n / (ms / 1e3) / 1e9}
    print(json.dumps(row), flush=True)
    del X, W, H, W0, H0
    torch.cuda.empty_cache()

# nTT sweeps with BCD at every step (ntt_decompose_bcd) next to the MU sweep, configs 3 and 4
if len(sys.argv) > 3 and sys.argv[3] == "sweep":
    for name in ("config3", "config4"):
        w = ni.workloads()[name]
        cores0 = torch.from_numpy(ni.make_cores(w.dims, w.ranks, w.seed).astype(np.float32)).cuda()
        A = torch.empty(w.numel, device="cuda")
        h.ntt_generate(w.dims, w.ranks, cores0, w.noise_amp, w.seed, ni.STREAM_NOISE, A)
        cores = torch.empty(P.cores_size(w.dims, w.ranks), device="cuda")
        row = {"workload": name, "iters_per_step": w.iters}
        for alg in ("bcd", "mu"):
            f = (lambda: h.ntt_decompose_bcd(A, w.dims, w.ranks, w.iters, w.seed, cores, want_error=True)) \
                if alg == "bcd" else \
                (lambda: h.ntt_decompose(A, w.dims, w.ranks, w.iters, w.seed, 1e-16, cores, want_error=True))
            f()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            err = f()
            e1.record()
            torch.cuda.synchronize()
            row[alg] = {"wall_ms": e0.elapsed_time(e1), "rel_err": err}
        print(json.dumps(row), flush=True)
        del A, cores
        torch.cuda.empty_cache()
