"""f2 + f3 + f4 at the paper's scale: the eps-driven nTT (Alg. 2 with the rank rule, MU 100
iterations per step) and the TT-SVD baseline on a 256^4 tensor whose train has
graded bond directions (ntt_inputs.make_cores_decay, TT ranks 10, rho 0.6, no noise); ranks capped
at 16.  Step 2 of both has min(m, n) = 256 r_1 > 512, i.e. the grid-wide eigensolver.  Tools only."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
dims, tr = [256] * 4, [10, 10, 10]
cores0 = torch.from_numpy(ni.make_cores_decay(dims, tr, 0.6, 0).astype(np.float32)).cuda()
A = torch.empty(256 ** 4, device="cuda")
h.ntt_generate(dims, tr, cores0, 0.0, 0, ni.STREAM_NOISE, A)
cap = P.cores_size(dims, [16] * 3)
cores = torch.empty(cap, device="cuda")
print("| eps | nTT ranks | nTT compression | nTT rel. error | nTT s | TT-SVD ranks | TT-SVD compression | TT-SVD rel. error | TT-SVD s |")
print("|---|---|---|---|---|---|---|---|---|")
for eps in (0.2, 0.1, 0.05, 0.02, 0.01):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rn, en = h.ntt_decompose_eps(A, dims, eps, 100, 0, 1e-16, cores, cap, max_ranks=[16] * 3, want_error=True)
    torch.cuda.synchronize()
    tn = time.perf_counter() - t0
    t0 = time.perf_counter()
    rs, es = h.ntt_tt_svd(A, dims, eps, cores, cap, max_ranks=[16] * 3, want_error=True)
    torch.cuda.synchronize()
    ts = time.perf_counter() - t0
    print(f"| {eps} | {rn} | {P.ntt_compression_ratio(dims, rn):.0f} | {en:.5f} | {tn:.2f} | {rs} | "
          f"{P.ntt_compression_ratio(dims, rs):.0f} | {es:.5f} | {ts:.2f} |", flush=True)
