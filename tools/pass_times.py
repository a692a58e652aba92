"""Per-pass durations of one persistent MU launch (NTT_PERSIST_TRACE stamps of CTA 0): pass 0 =
prologue (acc only, writes the X16 cache), passes 1..iters-1 = update + acc, pass iters = update
only.  Usage: python tools/pass_times.py m n r iters.  Tools only."""
import os
import sys

os.environ["NTT_PERSIST_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402
from paper_2008_01340_b200._lib import lib  # noqa: E402

m, n, r, it = (int(a) for a in sys.argv[1:5])
h = P.Handle(0)
X = torch.rand(m * n, device="cuda")
W = torch.rand(m * r, device="cuda")
H = torch.rand(r * n, device="cuda")
h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
torch.cuda.synchronize()
tr = lib().ntt_debug_persist_trace(h._h)
a = np.array([tr[i] for i in range(4 * (it + 1))], dtype=np.float64).reshape(it + 1, 4)
for p in range(it + 1):
    end = a[p + 1, 0] if p < it else float("nan")
    print(f"pass {p}: tiles {(a[p, 1] - a[p, 0]) / 1e3:.1f} us, to next pass start {(end - a[p, 0]) / 1e3:.1f} us")
