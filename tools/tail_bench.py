"""Small-unfolding MU timing (config 3 steps 3-5, config 4 tail steps): default plan vs NTT_NO_TINY,
100 iterations per call, CUDA events around the call (tools only, not the bench)."""
import json
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402

SHAPES = [(256, 32, 8), (256, 64, 8), (256, 128, 8), (256, 192, 8), (128, 256, 8), (64, 700, 8),
          (256, 1024, 8), (256, 32768, 8), (30, 216, 5), (30, 1296, 5), (30, 7776, 5), (5, 120, 4)]
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 100
h = P.Handle(0)


def t_call(X, m, n, r, W, H):
    h.ntt_nmf_mu(X, m, n, n, r, iters, 1e-16, W, H)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(3):
        e0.record()
        h.ntt_nmf_mu(X, m, n, n, r, iters, 1e-16, W, H)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for (m, n, r) in SHAPES:
    X = torch.rand(m * n, device="cuda")
    W = torch.rand(m * r, device="cuda")
    H = torch.rand(r * n, device="cuda")
    row = {"m": m, "n": n, "r": r}
    row["default_ms"] = t_call(X, m, n, r, W.clone(), H.clone())
    os.environ["NTT_NO_TINY"] = "1"
    row["no_tiny_ms"] = t_call(X, m, n, r, W.clone(), H.clone())
    del os.environ["NTT_NO_TINY"]
    print(json.dumps(row), flush=True)
