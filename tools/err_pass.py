"""Time of the Eq. 3 error pass (ntt_reconstruct with a reference, config-3 sizes; tools only)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
dims, ranks = [32] * 6, [8] * 5
cores = torch.from_numpy(ni.make_cores(dims, ranks, seed=0).astype(np.float32)).cuda()
A = torch.rand(32 ** 6, device="cuda")
for _ in range(3):
    h.ntt_reconstruct(dims, ranks, cores, ref=A, want_error=True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    h.ntt_reconstruct(dims, ranks, cores, ref=A, want_error=True)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print(f"error pass {ms:.3f} ms = {4 * 32 ** 6 / ms / 1e9:.2f} TB/s")
h.ntt_profile_enable(True)
for _ in range(10):
    h.ntt_reconstruct(dims, ranks, cores, ref=A, want_error=True)
torch.cuda.synchronize()
for l in range(0, 8):
    k, kms, by = h.ntt_profile_get(3, l)
    if k:
        print(f"stream kernel (class 3, level {l}): {kms / k:.3f} ms per launch = {by / (kms / 1e3) / 1e12:.2f} TB/s")
