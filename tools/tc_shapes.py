"""Per-iteration time of ntt_nmf_mu on tall tensor-core shapes, with the per-class profile (tools only)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
names = ["xstream", "xht", "wupdate", "ttstream", "other", "hpass2", "tc_xht", "tc_wtx"]
for (m, n, r, it) in [(1024, 1 << 21, 20, 10), (10240, 32768, 30, 10), (32768, 65536, 32, 5), (4096, 4096, 16, 20)]:
    X = torch.rand(m * n, device="cuda")
    W = torch.rand(m * r, device="cuda")
    H = torch.rand(r * n, device="cuda")
    h.ntt_nmf_mu(X, m, n, n, r, 2, 1e-16, W, H)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
    e1.record()
    torch.cuda.synchronize()
    h.ntt_profile_enable(True)
    h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
    prof = {names[c]: round(h.ntt_profile_get(c)[1] * 1e3 / it, 1) for c in range(8) if h.ntt_profile_get(c)[0]}
    h.ntt_profile_enable(False)
    print(f"{m}x{n} r{r}: {e0.elapsed_time(e1) * 1e3 / it:.1f} us/it  {prof}", flush=True)
    del X, W, H
    torch.cuda.empty_cache()
