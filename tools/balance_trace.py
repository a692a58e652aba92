"""Per-CTA pass timing of the persistent fused kernel (load-balance diagnostics; tools only)."""
import os
import sys

os.environ["NTT_PERSIST_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402
from paper_2008_01340_b200._lib import lib  # noqa: E402

h = P.Handle(0)
for (m, n, r) in [(256, 32**4, 8), (32, 32**5, 8)]:
    X = torch.rand(m * n, device="cuda")
    W = torch.rand(m * r, device="cuda")
    H = torch.rand(r * n, device="cuda")
    h.ntt_nmf_mu(X, m, n, n, r, 3, 1e-16, W, H)
    torch.cuda.synchronize()
    tr = lib().ntt_debug_persist_trace(h._h)
    g = 296 if m > 40 else 148
    end = np.array([tr[16384 + c] for c in range(g)], dtype=np.float64)
    st = np.array([tr[17408 + c] for c in range(g)], dtype=np.float64)
    dur = (end - st) / 1e3
    print(f"{m}x{n}: pass-1 duration per CTA us: min {dur.min():.1f} median {np.median(dur):.1f} max {dur.max():.1f}")
    print("  start spread us:", (st.max() - st.min()) / 1e3, " end spread us:", (end.max() - end.min()) / 1e3)
    order = np.argsort(dur)
    print("  slowest CTAs:", order[-12:].tolist(), " fastest:", order[:12].tolist())
    if g == 296:
        a, b = dur[:148], dur[148:]
        print(f"  CTA 0-147 median {np.median(a):.1f}, CTA 148-295 median {np.median(b):.1f}")
        print("  per-CTA dur (first 20):", np.round(dur[:20], 1).tolist())
    del X, W, H
