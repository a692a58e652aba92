"""Per-step timing of the BCD NMF on the unfolding shapes of config 3 (tools only)."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402
h = P.Handle(0)
for (m, n, r) in [(32, 32 ** 5, 8), (256, 32 ** 4, 8), (256, 32 ** 3, 8), (256, 1024, 8), (256, 32, 8)]:
    X = torch.rand(m * n, device="cuda") + 0.1
    W0 = torch.rand(m * r, device="cuda")
    H0 = torch.rand(r * n, device="cuda")
    for alg in ("bcd", "mu"):
        W, H = W0.clone(), H0.clone()
        f = (lambda: h.ntt_nmf_bcd(X, m, n, n, r, 100, W, H)) if alg == "bcd" else \
            (lambda: h.ntt_nmf_mu(X, m, n, n, r, 100, 1e-16, W, H))
        f()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        print(f"{alg} {m}x{n} r{r}: {e0.elapsed_time(e1):.2f} ms / 100 it", flush=True)
    del X, W, H, W0, H0
    torch.cuda.empty_cache()
