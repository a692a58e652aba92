import os, sys
import numpy as np, torch
sys.path.insert(0, ".")
import ntt_inputs as ni, oracle
import paper_2008_01340_b200 as P
oracle.build()
h = P.Handle(0)
def rel(a, b): return np.linalg.norm(a - b) / np.linalg.norm(b)
for (m, n, r) in [(256, 1024, 12), (64, 1024, 12), (32, 512, 16), (256, 1024, 8), (64, 1024, 9)]:
    for cs in ["", "16"]:
        if cs: os.environ["NTT_CLU_CS"] = cs
        else: os.environ.pop("NTT_CLU_CS", None)
        rng = np.random.default_rng(1)
        X = (rng.random((m, n)) * 4).astype(np.float32)
        W0 = ni.uniform(m * r, 1, 0x202).reshape(m, r).astype(np.float32)
        H0 = ni.uniform(r * n, 1, 0x203).reshape(r, n).astype(np.float32)
        out = []
        for it in (1, 2, 5):
            Wd, Hd = torch.from_numpy(W0).cuda(), torch.from_numpy(H0).cuda()
            h.ntt_nmf_mu(torch.from_numpy(X).cuda(), m, n, n, r, it, 1e-16, Wd, Hd)
            Wo, Ho = oracle.nmf_mu(X.astype(np.float64), W0.astype(np.float64), H0.astype(np.float64), it, eps=1e-16)
            out.append(f"it{it}: W {rel(Wd.cpu().numpy(), Wo):.1e} H {rel(Hd.cpu().numpy(), Ho):.1e}")
        print(m, n, r, "cs", cs or "auto", "path", h.mu_path(m, n, r), " | ".join(out), flush=True)
