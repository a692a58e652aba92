import sys, torch
sys.path.insert(0, ".")
import paper_2008_01340_b200 as P
h = P.Handle(0)
names = ["xstream", "xht", "wupdate", "ttstream", "other", "hpass2", "tc_xht", "tc_wtx"]
for (m, n, r) in [(15360, 64, 40), (3000, 200, 20)]:
    X = torch.rand(m * n, device="cuda"); W = torch.rand(m * r, device="cuda"); H = torch.rand(r * n, device="cuda")
    h.ntt_nmf_mu(X, m, n, n, r, 3, 1e-16, W, H)
    h.ntt_profile_enable(True)
    h.ntt_nmf_mu(X, m, n, n, r, 20, 1e-16, W, H)
    print(m, n, r, {names[c]: round(h.ntt_profile_get(c)[1] * 1e3 / 20, 1) for c in range(8) if h.ntt_profile_get(c)[0]})
    h.ntt_profile_enable(False)
