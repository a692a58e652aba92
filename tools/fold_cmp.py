import os, sys, json, torch
sys.path.insert(0, ".")
import paper_2008_01340_b200 as P
h = P.Handle(0)
g = torch.Generator(device="cuda"); g.manual_seed(1)
for (m, n, r) in [(32, 1 << 20, 8), (6, 1 << 18, 5)]:
    W0 = torch.rand(m, r, device="cuda", generator=g); H0 = torch.rand(r, n, device="cuda", generator=g)
    X = (W0 @ H0 + 0.1 * torch.rand(m, n, device="cuda", generator=g)).contiguous()
    Wi = torch.rand(m, r, device="cuda", generator=g); Hi = torch.rand(r, n, device="cuda", generator=g)
    W = Wi.clone(); H = Hi.clone()
    tr = h.ntt_nmf_bcd(X, m, n, n, r, 12, W, H, trace=True)
    print(os.environ.get("NTT_BCD_NO_FOLD", "fold"), m, n, r, json.dumps([round(t, 6) for t in tr]))
