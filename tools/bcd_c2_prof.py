"""BCD on config 2's shape (4096 x 4096, r 16): a few iterations for an ncu launch list (tools only)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402
h = P.Handle(0)
m = n = 4096
r = 16
X = torch.rand(m * n, device="cuda") + 0.1
W = torch.rand(m * r, device="cuda")
H = torch.rand(r * n, device="cuda")
h.ntt_nmf_bcd(X, m, n, n, r, 3, W, H)
torch.cuda.synchronize()
