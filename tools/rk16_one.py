"""One persistent k_fused_c<256, 8, 16> launch (256 x 2^22, r = 10, the paper's 256^4 step-1 class at a
quarter of its width) for an `ncu --set full -k regex:k_fused_c` capture (tools only).
    python tools/rk16_one.py [iters]"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
it = int(sys.argv[1]) if len(sys.argv) > 1 else 5
m, n, r = 256, 1 << 22, 10
X = torch.rand(m * n, device="cuda")
W = torch.rand(m * r, device="cuda")
H = torch.rand(r * n, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
e0.record()
h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / it
print(f"{m} x {n} r {r}: {ms:.3f} ms per iteration, {4.0 * n * (m + 2 * r) / (ms * 1e-3) / 1e9:.0f} GB/s algorithmic")
assert bool(torch.isfinite(W).all()) and bool(torch.isfinite(H).all())
