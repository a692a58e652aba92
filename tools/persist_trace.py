"""Phase timing of the persistent fused MU kernel (NTT_PERSIST_TRACE=1; tools only)."""
import os
import sys

os.environ["NTT_PERSIST_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402
from paper_2008_01340_b200._lib import lib  # noqa: E402

shapes = [(int(a), int(b), int(c), int(d)) for a, b, c, d in (x.split(',') for x in sys.argv[1:])] or \
    [(32, 32**5, 8, 20), (256, 32**4, 8, 20), (256, 32**3, 8, 50), (256, 32**2, 8, 50), (256, 32, 8, 50),
     (6, 6**9, 5, 20), (30, 6**4, 5, 50)]
h = P.Handle(0)
for (m, n, r, it) in shapes:
    X = torch.rand(m * n, device="cuda")
    W = torch.rand(m * r, device="cuda")
    H = torch.rand(r * n, device="cuda")
    h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
    e1.record()
    torch.cuda.synchronize()
    tot = e0.elapsed_time(e1) * 1e3 / it
    tr = lib().ntt_debug_persist_trace(h._h)
    a = np.array([tr[i] for i in range(4 * (it + 1))], dtype=np.float64).reshape(it + 1, 4)
    # per pass p >= 1: pass (stamp0 -> stamp1), barrier1 (1->2), slice+barrier2 (2->3), W update + next start (3 -> next 0)
    ps = a[1:-1]
    nxt = a[2:, 0]
    passt = np.median(ps[:, 1] - ps[:, 0]) / 1e3
    b1 = np.median(ps[:, 2] - ps[:, 1]) / 1e3
    b2 = np.median(ps[:, 3] - ps[:, 2]) / 1e3
    wu = np.median(nxt - ps[:, 3]) / 1e3
    f = np.array([tr[12288 + i] for i in range(4 * (it + 1))], dtype=np.float64).reshape(it + 1, 4)[1:-1]
    q = np.median(f[:, 0] - ps[:, 3]) / 1e3
    wupd = np.median(f[:, 1] - f[:, 0]) / 1e3
    gram = np.median(f[:, 2] - f[:, 1]) / 1e3
    tail = np.median(f[:, 3] - f[:, 2]) / 1e3
    nx = np.median(nxt - f[:, 3]) / 1e3
    cy = np.array([tr[8192 + i] for i in range(4 * (it + 1))], dtype=np.float64).reshape(it + 1, 4)[1:-1]
    print("   clock64 cycles: W update", np.median(cy[:, 1] - cy[:, 0]), "Gram", np.median(cy[:, 2] - cy[:, 1]))
    g = min((n + 127) // 128, 148 if m <= 40 else (148 if (m > 128 and r > 8) else 296))
    st1 = np.array([tr[17408 + i] for i in range(min(g, 1024))], dtype=np.float64)
    en1 = np.array([tr[16384 + i] for i in range(min(g, 1024))], dtype=np.float64)
    ok = (st1 > 0) & (en1 > 0)
    if ok.sum() > 1:
        d = (en1[ok] - st1[ok]) / 1e3
        e = (en1[ok] - en1[ok].min()) / 1e3
        print(f"   pass-1 per-CTA ({ok.sum()} CTAs) duration us: min {d.min():.1f} p50 {np.median(d):.1f} "
              f"max {d.max():.1f}; end spread p50 {np.median(e):.1f} p90 {np.percentile(e, 90):.1f} max {e.max():.1f}")
    print(f"{m}x{n} r{r}: {tot:.2f} us/iter | pass {passt:.2f} barrier1 {b1:.2f} slice+barrier2 {b2:.2f} "
          f"Wupdate->next {wu:.2f} us [Q load {q:.2f}, W update {wupd:.2f}, Gram {gram:.2f}, Wout {tail:.2f}, "
          f"-> next pass {nx:.2f}]", flush=True)
    del X, W, H
