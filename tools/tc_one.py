import sys, torch
sys.path.insert(0, ".")
import paper_2008_01340_b200 as P
h = P.Handle(0)
m, n, r = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (1024, 1 << 21, 20)
X = torch.rand(m * n, device="cuda"); W = torch.rand(m * r, device="cuda"); H = torch.rand(r * n, device="cuda")
h.ntt_nmf_mu(X, m, n, n, r, 3, 1e-16, W, H)
torch.cuda.synchronize()
