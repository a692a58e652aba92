"""Probe for the ncu LaunchFailed on graph-captured k_tiny (tools only): one config-1-shaped
nTT decomposition (graph on unless NTT_GRAPH=0), run under ncu by the caller."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import oracle  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
dims, ranks = [5, 4, 5, 6], [4, 3, 2]
A = oracle.tt_full_f32(dims, ranks, ni.make_cores(dims, ranks, seed=0))
Ad = torch.from_numpy(A).cuda()
cores = torch.empty(P.cores_size(dims, ranks), dtype=torch.float32, device="cuda")
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    h.ntt_decompose(Ad, dims, ranks, 10, 0, 1e-16, cores)
torch.cuda.synchronize()
print("ok", float(cores.sum()))
