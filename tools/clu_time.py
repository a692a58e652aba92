"""Per-iteration time of ntt_nmf_mu on the tail-step shapes, cluster mode vs the previous path
(NTT_NO_CLUSTER=1), CUDA events around one call of `it` iterations (tools only)."""
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402

shapes = [(256, 1024, 8), (256, 32, 8), (256, 40, 8), (256, 128, 8), (256, 256, 8), (100, 60, 5), (128, 32, 8), (30, 7776, 5), (30, 1296, 5), (30, 216, 5), (30, 36, 5),
          (256, 1024, 10), (256, 2048, 8), (64, 4096, 8), (128, 1024, 16), (20, 30, 4), (12, 5, 3)]
h = P.Handle(0)
for (m, n, r) in shapes:
    X = torch.rand(m * n, device="cuda")
    row = []
    for mode in ("cluster", "previous"):
        if mode == "previous":
            os.environ["NTT_NO_CLUSTER"] = "1"
        else:
            os.environ.pop("NTT_NO_CLUSTER", None)
        path = h.mu_path(m, n, r)
        W = torch.rand(m * r, device="cuda")
        H = torch.rand(r * n, device="cuda")
        it = 300
        h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
        e1.record()
        torch.cuda.synchronize()
        row.append(f"{mode} (path {path}) {e0.elapsed_time(e1) * 1e3 / it:.2f} us/it")
    print(f"{m}x{n} r{r}: " + " | ".join(row), flush=True)
os.environ.pop("NTT_NO_CLUSTER", None)
