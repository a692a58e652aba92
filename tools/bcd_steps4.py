"""Per-step BCD vs MU timing on config 4's unfolding shapes (tools only)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402
h = P.Handle(0)
for (m, n, r) in [(6, 6 ** 9, 5), (30, 6 ** 8, 5), (30, 6 ** 7, 5), (30, 6 ** 6, 5), (30, 6 ** 5, 5), (30, 6 ** 4, 5)]:
    X = torch.rand(m * n, device="cuda") + 0.1
    W0 = torch.rand(m * r, device="cuda")
    H0 = torch.rand(r * n, device="cuda")
    for alg in ("bcd", "mu"):
        W, H = W0.clone(), H0.clone()
        f = (lambda: h.ntt_nmf_bcd(X, m, n, n, r, 300, W, H)) if alg == "bcd" else \
            (lambda: h.ntt_nmf_mu(X, m, n, n, r, 300, 1e-16, W, H))
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        print(f"{alg} {m}x{n} r{r}: {e0.elapsed_time(e1):.2f} ms / 300 it", flush=True)
