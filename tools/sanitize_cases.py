"""Small invocations of every kernel class, for compute-sanitizer (memcheck / racecheck / synccheck).
Usage: compute-sanitizer --tool racecheck python tools/sanitize_cases.py"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import ntt_inputs as ni  # noqa: E402
import paper_2008_01340_b200 as P  # noqa: E402

h = P.Handle(0)


def mu(m, n, r, iters=3, what=""):
    rng = np.random.default_rng(m + n + r)
    X = torch.from_numpy(rng.random((m, n), dtype=np.float32)).cuda()
    W = torch.from_numpy(ni.uniform(m * r, 0, 0x202).astype(np.float32)).cuda()
    H = torch.from_numpy(ni.uniform(r * n, 0, 0x203).astype(np.float32)).cuda()
    h.ntt_nmf_mu(X, m, n, n, r, iters, 1e-16, W, H)
    torch.cuda.synchronize()
    assert torch.isfinite(W).all() and torch.isfinite(H).all(), what
    print("ok", what, m, n, r, flush=True)


def bcd(m, n, r, iters=3, what=""):
    rng = np.random.default_rng(m + n + r)
    X = torch.from_numpy(rng.random((m, n), dtype=np.float32)).cuda()
    W = torch.from_numpy(ni.uniform(m * r, 0, 0x202).astype(np.float32)).cuda()
    H = torch.from_numpy(ni.uniform(r * n, 0, 0x203).astype(np.float32)).cuda()
    h.ntt_nmf_bcd(X, m, n, n, r, iters, W, H)
    torch.cuda.synchronize()
    print("ok bcd", what, m, n, r, flush=True)


mu(5, 120, 4, what="k_tiny")
mu(8, 4096, 4, what="k_fused (FFMA, direct H)")
mu(40, 1024, 8, what="k_fused (FFMA, staged H)")
mu(32, 4096, 8, what="k_fused_m (tensor cores, X16 cache)")
mu(64, 2048, 8, what="k_fused_c<128> (tensor cores, X16 cache)")
mu(256, 1024, 8, what="k_fused_c<256>")
mu(300, 512, 16, what="k_skinny_tc16 2-pass")
mu(100, 700, 16, what="generic 2-pass")
bcd(32, 1024, 8, what="one-pass BCD with the H_m fold")
bcd(256, 1024, 8, what="one-pass BCD k_fused_c")
bcd(300, 512, 16, what="BCD tensor-core passes")
dims, ranks = [5, 4, 5, 6], [4, 3, 2]
A = torch.rand(int(np.prod(dims)), device="cuda")
cores = torch.empty(P.cores_size(dims, ranks), device="cuda")
e = h.ntt_decompose(A, dims, ranks, 3, 0, 1e-16, cores, want_error=True)
print("ok decompose + Eq. 3 error", e, flush=True)
ranks2, c2 = None, torch.empty(4096, device="cuda")
h.ntt_tt_svd(A, dims, 0.1, c2, 4096)
print("ok tt_svd", flush=True)
