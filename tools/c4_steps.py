"""Per-iteration time of the config-4 TT-step shapes through ntt_nmf_mu (tools only)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
for (m, n, r, it) in [(6, 6**9, 5, 60), (30, 6**8, 5, 100), (30, 6**7, 5, 200), (30, 6**6, 5, 300), (30, 6**5, 5, 300)]:
    X = torch.rand(m * n, device="cuda")
    W = torch.rand(m * r, device="cuda")
    H = torch.rand(r * n, device="cuda")
    h.ntt_nmf_mu(X, m, n, n, r, 5, 1e-16, W, H)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
    e1.record()
    torch.cuda.synchronize()
    print(f"{m}x{n} r{r} path {h.mu_path(m, n, r)}: {e0.elapsed_time(e1) * 1e3 / it:.1f} us/it", flush=True)
    del X, W, H
