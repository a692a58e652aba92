"""Cost of the cross-GPU reduction on a 1-rank distributed handle (config 3 nTT): single-GPU
handle vs ntt_create_dist with the in-kernel exchange (mode 1) vs the per-pass ncclAllReduce
path (mode 0).  With one rank the exchange stores go to the local buffer, so the difference to
the single-GPU handle is the protocol's own cost (push, flags, extra grid barrier); NVLink adds
its latency on a real multi-GPU box.  Per-step times from the library profiler.  Tools only."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

w = ni.workloads()["config3"]
h1 = P.Handle(0)
hd = P.Handle(0, unique_id=P.ntt_get_unique_id(), nranks=1, rank=0)
cores0 = torch.from_numpy(ni.make_cores(w.dims, w.ranks, w.seed).astype(np.float32)).cuda()
A = torch.empty(w.numel, device="cuda")
h1.ntt_generate(w.dims, w.ranks, cores0, w.noise_amp, w.seed, ni.STREAM_NOISE, A)
cores = torch.empty(P.cores_size(w.dims, w.ranks), device="cuda")
out = {}
for name, h, mode in (("single", h1, None), ("dist1_peer", hd, 1), ("dist1_nccl", hd, 0)):
    if mode is not None:
        h.ntt_set_dist_exchange(mode)
    for _ in range(2):
        h.ntt_decompose(A, w.dims, w.ranks, w.iters, w.seed, 1e-16, cores)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        h.ntt_decompose(A, w.dims, w.ranks, w.iters, w.seed, 1e-16, cores)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    h.ntt_profile_enable(True)
    h.ntt_decompose(A, w.dims, w.ranks, w.iters, w.seed, 1e-16, cores)
    h.ntt_profile_enable(True)
    h.ntt_decompose(A, w.dims, w.ranks, w.iters, w.seed, 1e-16, cores)
    steps = {}
    for l in range(1, len(w.dims)):
        steps[l] = round(sum(h.ntt_profile_get(c, l)[1] for c in range(8)), 3)
    h.ntt_profile_enable(False)
    out[name] = {"ms": round(ms, 3), "per_step_ms": steps}
    print(name, json.dumps(out[name]), flush=True)
print("exchanges on the dist handle:", hd.peer_exchange_count)
