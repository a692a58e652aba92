"""Config 2 (4096 x 4096, r 16) MU: per-kernel-class launches and time per iteration (tools only)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
m = n = 4096
r = 16
it = 50
dims, ranks, cores = ni.make_factor_cores(m, n, r, 0)
X = torch.empty(m * n, device="cuda")
h.ntt_generate(dims, ranks, torch.from_numpy(cores.astype(np.float32)).cuda(), 0.01, 0, ni.STREAM_NOISE, X)
W = torch.rand(m * r, device="cuda")
H = torch.rand(r * n, device="cuda")
h.ntt_nmf_mu(X, m, n, n, r, 3, 1e-16, W, H)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
e1.record()
torch.cuda.synchronize()
print("ms/iter (no profiler)", e0.elapsed_time(e1) / it)
h.ntt_profile_enable(True)
h.ntt_nmf_mu(X, m, n, n, r, it, 1e-16, W, H)
names = ["xstream", "xht", "wupdate", "ttstream", "other", "hpass2", "tc_xht", "tc_wtx"]
out = {}
for c in range(8):
    k, ms, by = h.ntt_profile_get(c)
    if k:
        out[names[c]] = {"launches_per_iter": k / it, "us_per_iter": 1e3 * ms / it}
print(json.dumps(out))
