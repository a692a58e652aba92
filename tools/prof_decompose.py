"""Per-TT-step breakdown of one ntt_decompose (device-generated synthetic input)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "config3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
w = ni.workloads()[name]
h = P.Handle(0)
cores0 = torch.from_numpy(ni.make_cores(w.dims, w.ranks, 0).astype(np.float32)).cuda()
A = torch.empty(w.numel, device="cuda")
h.ntt_generate(w.dims, w.ranks, cores0, w.noise_amp, 0, ni.STREAM_NOISE, A)
cores = torch.empty(P.cores_size(w.dims, w.ranks), device="cuda")
err = h.ntt_decompose(A, w.dims, w.ranks, w.iters, 0, 1e-16, cores, want_error=True)
torch.cuda.synchronize()
h.ntt_profile_enable(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    err = h.ntt_decompose(A, w.dims, w.ranks, w.iters, 0, 1e-16, cores, want_error=True)
e1.record()
torch.cuda.synchronize()
tot = e0.elapsed_time(e1) / reps
names = ["xstream", "xht", "wupdate", "ttstream", "other", "hpass2"]
d = len(w.dims)
print(json.dumps({"workload": name, "ms_per_decompose": tot, "rel_err": err}))
for l in range(0, d + 1):
    row = {}
    for c in range(6):
        k, ms, by = h.ntt_profile_get(c, l)
        if k:
            row[names[c]] = [k // reps, round(ms / reps, 3), round(by / (ms / 1e3) / 1e9, 1) if ms > 0 else None]
    if row:
        print(f"step {l}: " + json.dumps(row))
