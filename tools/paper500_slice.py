"""The paper's 500 GB tensor (1024 x 512^3, TT ranks 1,20,30,40,1) -- one GPU's share of the
8-GPU run (SURVEY s.8(f3)): the rank-0 block of the last mode, 1024 x 512 x 512 x 64 (68.7 GB fp32),
generated on the device from a random non-negative TT of those ranks (+ 1 % uniform noise), then the
fixed-rank MU nTT (100 iterations per step) with its Eq. 3 error and per-step kernel profile.  This is
the per-GPU compute of the 8-GPU run without the cross-GPU exchange (DESIGN.md s.7).  Tools only:
python tools/paper500_slice.py > profiles/paper500_slice_r2.json"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

gdims, ranks, iters, p = [1024, 512, 512, 512], [20, 30, 40], 100, 8
dims = gdims[:-1] + [gdims[-1] // p]
cores_g = ni.make_cores(gdims, ranks, 0)
last = cores_g[-ranks[-1] * gdims[-1]:].reshape(ranks[-1], gdims[-1])[:, : dims[-1]]
cores_l = np.concatenate([cores_g[: -ranks[-1] * gdims[-1]], last.ravel()]).astype(np.float32)
h = P.Handle(0)
N = int(np.prod(dims))
A = torch.empty(N, device="cuda")
noise = 0.01 * 0.5 ** 4 * 20 * 30 * 40  # 1 % of the mean entry (as configs 3 and paper256)
h.ntt_generate(dims, ranks, torch.from_numpy(cores_l).cuda(), noise, 0, ni.STREAM_NOISE, A)
cores = torch.empty(P.cores_size(dims, ranks), device="cuda")
free0, total = torch.cuda.mem_get_info()
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
h.ntt_profile_enable(True)
e0, e1 = ev(), ev()
e0.record()
err = h.ntt_decompose(A, dims, ranks, iters, 0, 1e-16, cores, want_error=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
names = ["xstream", "xht", "wupdate", "ttstream", "other", "hpass2", "tc_xht", "tc_wtx"]
prof = {}
for l in range(1, len(dims) + 1):
    row = {}
    for c in range(8):
        k, t, by = h.ntt_profile_get(c, l)
        if k:
            row[names[c]] = {"launches": k, "ms": round(t, 3), "GBps": round(by / (t * 1e6), 1) if t > 0 else 0.0}
    prof[f"step{l}" if l < len(dims) else "last_core+error"] = row
h.ntt_profile_enable(False)
free1, _ = torch.cuda.mem_get_info()
print(json.dumps({"workload": "paper500 rank-0 slice (P:461)", "global_dims": gdims, "local_dims": dims,
                  "ranks": ranks, "iters_per_step": iters, "input_GB": N * 4 / 1e9, "ntt_wall_ms": ms,
                  "note": "profiling on (events per launch); one decomposition incl. the Eq. 3 error pass",
                  "rel_error": err, "device_GB_used": (total - free1) / 1e9, "per_step": prof,
                  "mu_iter_per_s": 3 * iters / (ms / 1e3)}, indent=1))
