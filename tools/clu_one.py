"""One cluster-mode MU call (tools only; for ncu): python tools/clu_one.py m n r iters"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402

m, n, r, it = (int(a) for a in sys.argv[1:5])
h = P.Handle(0)
X = torch.rand(m * n, device="cuda")
W = torch.rand(m * r, device="cuda")
H = torch.rand(r * n, device="cuda")
h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
torch.cuda.synchronize()
print("path", h.mu_path(m, n, r))
