"""Phase cycles of the tiny-mode MU kernel (mu_tiny.cu; NTT_PERSIST_TRACE=1; tools only)."""
import os
import sys

os.environ["NTT_PERSIST_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402
from paper_2008_01340_b200._lib import lib  # noqa: E402

h = P.Handle(0)
for (m, n, r) in [(5, 120, 4), (16, 30, 3), (15, 6, 2), (30, 36, 5), (30, 6, 5)]:
    it = 60
    X = torch.rand(m * n, device="cuda")
    W = torch.rand(m * r, device="cuda")
    H = torch.rand(r * n, device="cuda")
    assert h.mu_path(m, n, r) == 1
    h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
    torch.cuda.synchronize()
    tr = lib().ntt_debug_persist_trace(h._h)
    a = np.array([tr[12288 + i] for i in range(8 * it)], dtype=np.float64).reshape(it, 8)[5:-1]
    nxt = np.array([tr[12288 + 8 * (i + 1)] for i in range(5, it - 1)], dtype=np.float64)
    d = [np.median(a[:, k + 1] - a[:, k]) for k in range(5)]
    tot = np.median(nxt - a[:, 0])
    print(f"{m}x{n} r{r}: {tot:.0f} cycles/it | P,Q {d[0]:.0f}, chunk sum {d[1]:.0f}, W update {d[2]:.0f}, "
          f"G {d[3]:.0f}, H update {d[4]:.0f}, loop {np.median(nxt - a[:, 5]):.0f}", flush=True)
