"""Eq. 3 error pass on the paper's 256^4 shape at TT ranks 10 (k_tt_err's RK = 16 class; tools only)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
dims, ranks = [256] * 4, [10] * 3
cores = torch.from_numpy(ni.make_cores(dims, ranks, seed=0).astype(np.float32)).cuda()
A = torch.rand(256 ** 4, device="cuda")
for _ in range(2):
    h.ntt_reconstruct(dims, ranks, cores, ref=A, want_error=True)
h.ntt_profile_enable(True)
for _ in range(5):
    h.ntt_reconstruct(dims, ranks, cores, ref=A, want_error=True)
torch.cuda.synchronize()
for l in range(0, 8):
    k, kms, by = h.ntt_profile_get(3, l)
    if k:
        print(f"256^4 r10 stream kernel: {kms / k:.3f} ms per launch = {by / (kms / 1e3) / 1e12:.2f} TB/s")
