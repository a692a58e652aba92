"""Single-NMF MU timing for BASELINE configs 2 and 5 (tools only, not the bench).

    python tools/bench_nmf.py [config2|config5] [iters]

Config 5 at 1 GPU runs on the 32768 x 65536 row slice (SURVEY s.8(d) d.2).
X = W0 H0 + noise is generated on the device by ntt_generate (a d = 2 train).
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

names = ["xstream", "xht", "wupdate", "ttstream", "other", "hpass2", "tc_xht", "tc_wtx"]
which = sys.argv[1:2] or ["config2", "config5"]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 10
h = P.Handle(0)
for name in (which if isinstance(which, list) else [which]):
    w = ni.workloads()[name]
    m, n = w.dims
    r = w.ranks[0]
    if name == "config5":
        m = 32768
    dims, ranks, cores = ni.make_factor_cores(m, n, r, 0)
    X = torch.empty(m * n, device="cuda")
    h.ntt_generate(dims, ranks, torch.from_numpy(cores.astype(np.float32)).cuda(), w.noise_amp or 0.01, 0,
                   ni.STREAM_NOISE, X)
    W = torch.empty(m * r, device="cuda")
    H = torch.empty(r * n, device="cuda")
    h.ntt_fill_uniform(W, m * r, 0, ni.stream_w(1))
    h.ntt_fill_uniform(H, r * n, 0, ni.stream_h(1))
    h.ntt_nmf_mu(X, m, n, n, r, 2, 1e-16, W, H)
    torch.cuda.synchronize()
    h.ntt_profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.ntt_nmf_mu(X, m, n, n, r, iters, 1e-16, W, H)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    alg2 = 4.0 * n * (2 * m + 3 * r) + 4.0 * 3 * m * r  # 2-pass algorithmic bytes / iteration
    row = {"workload": name, "m": m, "n": n, "r": r, "iters": iters, "ms_per_iter": ms,
           "mu_iter_per_s": 1e3 / ms, "eff_GBps_2pass": alg2 / (ms / 1e3) / 1e9,
           "flop_per_iter": 4.0 * m * n * r, "TFLOPs": 4.0 * m * n * r / (ms / 1e3) / 1e12}
    for c in range(8):
        k, t, by = h.ntt_profile_get(c)
        if k:
            row[names[c]] = {"launches": k, "us_each": 1e3 * t / k, "GBps": by / (t / 1e3) / 1e9 if t > 0 else 0}
    h.ntt_profile_enable(False)
    print(json.dumps(row), flush=True)
    del X, W, H
    torch.cuda.empty_cache()
