import sys, numpy as np, torch
sys.path.insert(0, ".")
import ntt_inputs as ni, paper_2008_01340_b200 as P
h = P.Handle(0)
w = ni.workloads()["config3"]
cores0 = torch.from_numpy(ni.make_cores(w.dims, w.ranks, w.seed).astype(np.float32)).cuda()
A = torch.empty(w.numel, device="cuda")
h.ntt_generate(w.dims, w.ranks, cores0, w.noise_amp, w.seed, ni.STREAM_NOISE, A)
cores = torch.empty(P.cores_size(w.dims, w.ranks), device="cuda")
h.ntt_decompose_bcd(A, w.dims, w.ranks, 5, w.seed, cores)
torch.cuda.synchronize()
