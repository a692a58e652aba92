"""k_fused_c rank-16 class (the paper's 256^4 step 1 shape class, r = 10): timing per pass at
256 x 2^22 and 256 x 2^24, r = 10 and r = 8 for contrast (tools only)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
it = int(sys.argv[1]) if len(sys.argv) > 1 else 20
for (m, n, r) in [(256, 1 << 22, 10), (256, 1 << 22, 8), (256, 1 << 22, 16), (256, 1 << 24, 10)]:
    X = torch.rand(m * n, device="cuda")
    W = torch.rand(m * r, device="cuda")
    H = torch.rand(r * n, device="cuda")
    h.ntt_nmf_mu(X, m, n, n, r, 2, 1e-16, W, H)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / it
    gbs = 4.0 * n * (m + 2 * r) / (ms * 1e-3) / 1e9
    print(f"{m} x {n} r {r}: {ms:.3f} ms per iteration, {gbs:.0f} GB/s algorithmic", flush=True)
    del X, W, H
    torch.cuda.empty_cache()
