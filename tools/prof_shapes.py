"""Per-shape MU timing via the library's event profiler (tools only, not the bench)."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402

SHAPES = [(32, 32**5, 8), (256, 32**4, 8), (256, 32**3, 8), (256, 32**2, 8), (256, 32, 8),
          (6, 6**9, 5), (30, 6**8, 5), (30, 6**7, 5), (30, 6**6, 5), (30, 6**3, 5)]
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
h = P.Handle(0)
names = ["xstream", "xht", "wupdate", "ttstream", "other", "hpass2"]
out = []
for (m, n, r) in SHAPES:
    X = torch.rand(m * n, device="cuda")
    W = torch.rand(m * r, device="cuda")
    H = torch.rand(r * n, device="cuda")
    h.ntt_nmf_mu(X, m, n, n, r, 3, 1e-16, W, H)
    torch.cuda.synchronize()
    h.ntt_profile_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.ntt_nmf_mu(X, m, n, n, r, iters, 1e-16, W, H)
    e1.record()
    torch.cuda.synchronize()
    tot = e0.elapsed_time(e1)
    row = {"m": m, "n": n, "r": r, "ms_per_iter": tot / iters}
    for c in range(6):
        k, ms, by = h.ntt_profile_get(c)
        if k:
            row[names[c]] = {"launches": k, "us_each": 1e3 * ms / k, "GBps": by / (ms / 1e3) / 1e9 if ms > 0 else 0}
    h.ntt_profile_enable(False)
    out.append(row)
    print(json.dumps(row), flush=True)
    del X, W, H
