"""BCD on the config-5 slice: a few iterations for an ncu launch list (tools only)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402
h = P.Handle(0)
w = ni.workloads()["config5"]
m, n, r = 32768, w.dims[1], w.ranks[0]
dims, ranks, cores = ni.make_factor_cores(m, n, r, 0)
X = torch.empty(m * n, device="cuda")
h.ntt_generate(dims, ranks, torch.from_numpy(cores.astype(np.float32)).cuda(), w.noise_amp or 0.01, 0, ni.STREAM_NOISE, X)
W = torch.empty(m * r, device="cuda")
H = torch.empty(r * n, device="cuda")
h.ntt_fill_uniform(W, m * r, 0, ni.stream_w(1))
h.ntt_fill_uniform(H, r * n, 0, ni.stream_h(1))
h.ntt_nmf_bcd(X, m, n, n, r, 3, W, H)
torch.cuda.synchronize()
