"""Is the per-CTA pass time of the persistent step-1 kernel systematic (same CTAs / SMs slow in
every pass)?  NTT_PERSIST_TRACE stamps; tools only."""
import os
import sys

os.environ["NTT_PERSIST_TRACE"] = "1"
import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402
from paper_2008_01340_b200._lib import lib  # noqa: E402

h = P.Handle(0)
for (m, n, r) in [(32, 32**5, 8), (6, 6**9, 5), (256, 32**4, 8)]:
    X = torch.rand(m * n, device="cuda")
    W = torch.rand(m * r, device="cuda")
    H = torch.rand(r * n, device="cuda")
    h.ntt_nmf_mu(X, m, n, n, r, 6, 1e-16, W, H)
    torch.cuda.synchronize()
    tr = lib().ntt_debug_persist_trace(h._h)
    g = min((n + 127) // 128, 148 if m <= 40 else 296)
    a = np.array([tr[i] for i in range(4 * 7)], dtype=np.float64).reshape(7, 4)
    st = [a[p, 0] for p in range(7)]  # CTA 0's pass starts (after barrier 2 of the previous pass)
    ends = [np.array([tr[16384 + c] for c in range(g)], dtype=np.float64)]
    for p in range(2, 5):
        ends.append(np.array([tr[18432 + 1024 * (p - 2) + c] for c in range(g)], dtype=np.float64))
    dur = [ends[p - 1] - st[p] for p in range(1, 5)]
    sm = np.array([tr[21504 + c] for c in range(g)])
    d = np.array(dur) / 1e3
    print(f"{m}x{n}: per-pass spread (max-min) us:", [f"{x.max() - x.min():.1f}" for x in d])
    cc = np.corrcoef(d)
    print("  correlation of per-CTA durations between passes:", np.round(cc[0, 1:], 2), np.round(cc[1, 2:], 2))
    mean = d.mean(axis=0)
    order = np.argsort(mean)
    print("  fastest CTAs (sm):", [(int(c), int(sm[c]), round(mean[c] - mean.min(), 1)) for c in order[:6]])
    print("  slowest CTAs (sm):", [(int(c), int(sm[c]), round(mean[c] - mean.min(), 1)) for c in order[-10:]])
    # by SM id group (tpc = sm // 2, 'gpc-ish' = sm // 18)
    for grp in (2, 16, 18, 20):
        gi = sm // grp
        means = [mean[gi == k].mean() for k in np.unique(gi)]
        print(f"  mean by smid//{grp}:", np.round(np.array(means) - min(means), 1))
    del X, W, H
