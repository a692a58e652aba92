"""One config-4 nTT decomposition (for ncu captures of its step-1 kernel; tools only)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402
h = P.Handle(0)
w = ni.workloads()["config4"]
cores0 = torch.from_numpy(ni.make_cores(w.dims, w.ranks, w.seed).astype(np.float32)).cuda()
A = torch.empty(w.numel, device="cuda")
h.ntt_generate(w.dims, w.ranks, cores0, w.noise_amp, w.seed, ni.STREAM_NOISE, A)
cores = torch.empty(P.cores_size(w.dims, w.ranks), device="cuda")
h.ntt_decompose(A, w.dims, w.ranks, w.iters, w.seed, 1e-16, cores)
torch.cuda.synchronize()
