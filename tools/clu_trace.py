"""Phase timing of the cluster-mode MU kernel (mu_cluster.cu; NTT_PERSIST_TRACE=1; tools only)."""
import os
import sys

os.environ["NTT_PERSIST_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402
from paper_2008_01340_b200._lib import lib  # noqa: E402

shapes = [(256, 1024, 8), (256, 256, 8), (30, 7776, 5), (30, 1296, 5), (128, 1024, 16), (64, 4096, 8)]
names = ["P,Q reduce", "W update", "Gram", "B1", "gather", "H update", "partials", "B2"]
h = P.Handle(0)
for (m, n, r) in shapes:
    it = 60
    X = torch.rand(m * n, device="cuda")
    W = torch.rand(m * r, device="cuda")
    H = torch.rand(r * n, device="cuda")
    assert h.mu_path(m, n, r) == 2
    h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
    torch.cuda.synchronize()
    tr = lib().ntt_debug_persist_trace(h._h)
    a = np.array([tr[12288 + i] for i in range(8 * it)], dtype=np.float64).reshape(it, 8)
    nxt = np.concatenate([a[1:, 0:1], a[:-1, 7:8]], axis=1)[:, 0]
    a = a[:-1]
    d = np.diff(a, axis=1)
    parts = [np.median(d[5:, k]) / 1e3 for k in range(7)] + [np.median(nxt[5:] - a[5:, 7]) / 1e3]
    tot = np.median(nxt[5:] - a[5:, 0]) / 1e3
    print(f"{m}x{n} r{r}: {tot:.2f} us/it | " + ", ".join(f"{nm} {v:.2f}" for nm, v in zip(names, parts)),
          flush=True)
