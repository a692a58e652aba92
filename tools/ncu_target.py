"""Small deterministic target for ncu: 2 MU iterations on config-3 step-1 and step-2 shapes."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2008_01340_b200 as P
h = P.Handle(0)
shapes = [(32, 32**5, 8), (256, 32**4, 8)]
if len(sys.argv) > 1:
    shapes = [shapes[int(a)] for a in sys.argv[1:]]
for (m, n, r) in shapes:
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.rand(m * n, device="cuda", generator=g)
    W = torch.rand(m * r, device="cuda", generator=g)
    H = torch.rand(r * n, device="cuda", generator=g)
    h.ntt_nmf_mu(X, m, n, n, r, 2, 1e-16, W, H)
    torch.cuda.synchronize()
    print(m, n, r, "done", float(W.sum()))
