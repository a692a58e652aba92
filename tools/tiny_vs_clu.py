"""Tiny mode (one CTA) vs cluster mode on the small TT-step shapes (tools only)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
for (m, n, r) in [(30, 216, 5), (30, 36, 5), (30, 6, 5), (5, 120, 4), (16, 30, 3), (15, 6, 2), (64, 180, 8),
                  (24, 400, 6)]:
    X = torch.rand(m * n, device="cuda")
    row = []
    for mode in ("tiny", "cluster"):
        if mode == "cluster":
            os.environ["NTT_NO_TINY"] = "1"
        else:
            os.environ.pop("NTT_NO_TINY", None)
        W = torch.rand(m * r, device="cuda")
        H = torch.rand(r * n, device="cuda")
        it = 300
        h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
        e1.record()
        torch.cuda.synchronize()
        row.append(f"{mode}(p{h.mu_path(m, n, r)}) {e0.elapsed_time(e1) * 1e3 / it:.2f}")
    print(m, n, r, " | ".join(row), flush=True)
os.environ.pop("NTT_NO_TINY", None)
