import os, sys
import torch
sys.path.insert(0, ".")
import paper_2008_01340_b200 as P
h = P.Handle(0)
for (m, n, r) in [(256, 32, 8), (256, 16, 8), (128, 32, 8), (100, 60, 5), (256, 64, 8)]:
    X = torch.rand(m * n, device="cuda")
    row = []
    for cs in ("none", "2", "4", "8"):
        if cs == "none": os.environ["NTT_NO_CLUSTER"] = "1"; os.environ.pop("NTT_CLU_CS", None)
        else: os.environ.pop("NTT_NO_CLUSTER", None); os.environ["NTT_CLU_CS"] = cs
        W = torch.rand(m * r, device="cuda"); H = torch.rand(r * n, device="cuda")
        it = 300
        h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H); e1.record(); torch.cuda.synchronize()
        row.append(f"{cs}(p{h.mu_path(m, n, r)}) {e0.elapsed_time(e1) * 1e3 / it:.2f}")
    print(m, n, r, " | ".join(row), flush=True)
