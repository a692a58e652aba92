"""eps sweep of the eps-driven nTT (Alg. 2 with the SVD rank rule) against the TT-SVD
baseline at the same eps (P:453's protocol: compression ratio Eq. 4 vs relative error Eq. 3), on
synthetic non-negative TT tensors whose unfolding spectra decay geometrically
(ntt_inputs.make_cores_decay: core entries U[0,1) x rho^(a+b)).  Also the U[0,1) train of round 1
for contrast.  Tools only (writes a markdown table to stdout)."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)
EPS = [0.5, 0.25, 0.125, 0.075, 0.05, 0.025, 0.01, 0.005, 0.001]
cases = [
    ("32^6 TT ranks 16, rho 0.7 (decaying)", [32] * 6, [16] * 5, 0.7, 100),
    ("32^4 TT ranks 16, rho 0.5 (decaying)", [32] * 4, [16] * 3, 0.5, 100),
    ("32^4 TT ranks (6,8,6), U[0,1) cores (flat spectrum after the mean)", [32] * 4, [6, 8, 6], 1.0, 100),
]
print("| tensor | eps | nTT ranks | nTT compression (Eq. 4) | nTT rel. error (Eq. 3) | nTT ms "
      "| TT-SVD ranks | TT-SVD compression | TT-SVD rel. error | TT-SVD ms |")
print("|---|---|---|---|---|---|---|---|---|---|")
for name, dims, tr, rho, iters in cases:
    cores0 = torch.from_numpy(ni.make_cores_decay(dims, tr, rho, 0).astype(np.float32)).cuda()
    N = int(np.prod(dims))
    A = torch.empty(N, device="cuda")
    h.ntt_generate(dims, tr, cores0, 0.0, 0, ni.STREAM_NOISE, A)
    capn = P.cores_size(dims, [64] * (len(dims) - 1))
    cores = torch.empty(capn, device="cuda")
    for e in EPS:
        try:
            h.ntt_decompose_eps(A, dims, e, 2, 0, 1e-16, cores, capn)  # warm-up
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ranks, err = h.ntt_decompose_eps(A, dims, e, iters, 0, 1e-16, cores, capn, want_error=True)
            torch.cuda.synchronize()
            ms = (time.perf_counter() - t0) * 1e3
            cr = P.ntt_compression_ratio(dims, ranks)
            nt = f"{ranks} | {cr:.1f} | {err:.5f} | {ms:.1f}"
        except Exception as ex:  # noqa: BLE001
            nt = f"({str(ex)[:60]}) | | |"
        try:
            h.ntt_tt_svd(A, dims, e, cores, capn)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rs, es = h.ntt_tt_svd(A, dims, e, cores, capn, want_error=True)
            torch.cuda.synchronize()
            ms2 = (time.perf_counter() - t0) * 1e3
            ts = f"{rs} | {P.ntt_compression_ratio(dims, rs):.1f} | {es:.5f} | {ms2:.1f}"
        except Exception as ex:  # noqa: BLE001
            ts = f"({str(ex)[:60]}) | | |"
        print(f"| {name} | {e} | {nt} | {ts} |", flush=True)
    del A, cores
