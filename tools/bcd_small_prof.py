"""BCD on a small unfolding (30 x 1296, r 5; config 4 step 6) for an ncu launch list (tools only)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402
h = P.Handle(0)
m, n, r = 30, 1296, 5
X = torch.rand(m * n, device="cuda") + 0.1
W = torch.rand(m * r, device="cuda")
H = torch.rand(r * n, device="cuda")
h.ntt_nmf_bcd(X, m, n, n, r, 4, W, H)
torch.cuda.synchronize()
