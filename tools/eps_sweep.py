"""eps sweep of the eps-driven nTT (Alg. 2 with the SVD rank rule): chosen
ranks, compression ratio (Eq. 4), relative error (Eq. 3) and wall time on synthetic
non-negative TT tensors (SURVEY s.8(f) f2, cf. the paper's Fig. 8 protocol P:453).
Tools only (writes a markdown table to stdout)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
cases = [
    ("32^4 TT ranks (6,8,6) + 1% noise", [32] * 4, [6, 8, 6], 0.01 * 6 * 8 * 6 / 8, 100, None,
     [0.5, 0.25, 0.125, 0.075, 0.01, 0.005]),
    ("config 3: 32^6 TT ranks 8 + 1% noise, max ranks 8", [32] * 6, [8] * 5, 5.12, 100, [8] * 5, [0.5, 0.2, 0.1, 0.05]),
]
print("| tensor | eps | ranks | compression (Eq. 4) | rel. error (Eq. 3) | nTT wall ms |")
print("|---|---|---|---|---|---|")
for name, dims, tr, noise, iters, cap, eps_list in cases:
    cores0 = torch.from_numpy(ni.make_cores(dims, tr, 0).astype(np.float32)).cuda()
    N = int(np.prod(dims))
    A = torch.empty(N, device="cuda")
    h.ntt_generate(dims, tr, cores0, noise, 0, ni.STREAM_NOISE, A)
    capn = P.cores_size(dims, cap if cap else [64] * (len(dims) - 1))
    cores = torch.empty(capn, device="cuda")
    for e in eps_list:
        h.ntt_decompose_eps(A, dims, e, 2, 0, 1e-16, cores, capn, max_ranks=cap)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ranks, err = h.ntt_decompose_eps(A, dims, e, iters, 0, 1e-16, cores, capn, max_ranks=cap, want_error=True)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        cr = P.ntt_compression_ratio(dims, ranks)
        print(f"| {name} | {e} | {ranks} | {cr:.1f} | {err:.4f} | {ms:.1f} |", flush=True)
    del A, cores
