"""Diagnostic: where does the BCD objective trace of the GPU (Gram identity, R25) differ from
the oracle's on config 2 (4096^2, r 16)?  Splits |obj_gpu - obj_ora| into the objective's
evaluation error (GPU trace vs the direct fp64 residual of the GPU's own factors) and the
trajectory difference (direct residual of GPU factors vs the oracle's)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import ntt_inputs as ni
import oracle as ora
import paper_2008_01340_b200 as P
from test_gpu_fullsize import _factor_input

m = n = 4096
r = 16
X = _factor_input(m, n, r, "absnormal")
W0 = ni.uniform(m * r, 0, ni.stream_w(1)).reshape(m, r).astype(np.float32)
H0 = ni.uniform(r * n, 0, ni.stream_h(1)).reshape(r, n).astype(np.float32)
h = P.Handle(0)
Xd = torch.from_numpy(X.ravel()).cuda()
Xdd = Xd.view(m, n).double()
xx = float((Xdd ** 2).sum())
for iters in (1, 5, 20, 50, 100):
    Wd, Hd = torch.from_numpy(W0.ravel().copy()).cuda(), torch.from_numpy(H0.ravel().copy()).cuda()
    trg = np.array(h.ntt_nmf_bcd(Xd, m, n, n, r, iters, Wd, Hd, trace=True))
    res = 0.5 * float(((Xdd - Wd.view(m, r).double() @ Hd.view(r, n).double()) ** 2).sum())
    Wo, Ho, tro = ora.nmf_bcd(X.astype(np.float64), W0, H0, iters, trace=True)
    print(f"iters {iters:4d}: obj/||X||^2 gpu-trace {trg[-1]/xx:.4e} gpu-direct {res/xx:.4e} oracle {tro[-1]/xx:.4e}"
          f" | eval err {abs(trg[-1]-res)/xx:.2e}  trajectory {abs(res-tro[-1])/xx:.2e}")
