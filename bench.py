#!/usr/bin/env python
"""bench.py -- MU-NMF nTT hot path on B200 (arXiv 2008.01340), BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload config3]

A step is one pass of the whole hot path (SURVEY s.8(a) rows a1-a7) over one
synthetic input: ntt_decompose (unfold, init, MU W/H half-steps, core emission,
sweep) plus the Eq. 3 relative error of the result.  Default workload: config 3
(32^6 fp32 = 4.29 GB > L2, TT ranks 8, 100 MU iterations per step -> 500 MU
iterations per decomposition), the largest BASELINE config the nTT sweep runs on
at 1 GPU.  Under torchrun (N > 1) the last tensor mode is block-partitioned over
the ranks (strong scaling, one NCCL all-reduce of the fp64 (XH^T, HH^T)
partials per MU pass).

Prints ONE JSON line (rank 0).  See DESIGN.md s.8 for the roofline bytes.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# what the paths compute in (R13): storage fp32 everywhere
ARITH_NTT = ("X.W and X.Hn^T products on warp-level tensor cores (mma.sync m16n8k16) as fp16 hi + lo splits of "
             "power-of-two-scaled operands (hi.hi + hi.lo + lo.hi, ~22 significant bits), fp32 accumulation within a "
             "tile, fp64 across tiles / CTAs / GPUs; m <= 16 unfoldings: fp32 FFMA; H update fp32; W update and "
             "Grams fp64 (k_fused_m / k_fused_c / k_fused)")
ARITH_TC = ("tcgen05 kind::f16 with fp16 hi + lo splits (~22 significant bits), fp32 TMEM accumulation flushed to "
            "fp64; W update fp64, H update fp32")
METRIC = "NMF-MU iterations/sec (nTT sweep, all d-1 steps; ntt wall time and HBM GB/s in roofline)"
UNIT = "MU-iter/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config3")
    ap.add_argument("--iters", type=int, default=None, help="override MU iterations per TT step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-other", action="store_true", help="skip the configs 1, 2, 4, 5 side measurements")
    ap.add_argument("--oracle-full", action="store_true",
                    help="time the oracle on the FULL config-4 nTT (minutes) instead of 3 iterations/step scaled")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rk = int(os.environ.get("RANK", "0"))
    lr = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rk, lr


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            return None
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "samples": len(sm), "reasons": sorted(reasons)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------ workload
def workload(name: str, iters_override=None):
    import ntt_inputs as ni
    w = ni.workloads()[name]
    if w.kind != "ntt":
        raise SystemExit(f"bench runs the nTT sweep; {name} is a single-NMF parity case")
    if iters_override:
        w.iters = iters_override
    return w


def step_shapes(dims, ranks):
    fr = [1, *ranks, 1]
    N = 1
    for x in dims:
        N *= x
    out, rest = [], N
    for l in range(1, len(dims)):
        rest //= dims[l - 1]
        out.append((fr[l - 1] * dims[l - 1], rest, fr[l]))
    return out


# ------------------------------------------------------------- oracle timing
def oracle_sample_time(dims, ranks, iters, budget_elems=1 << 25):
    """Oracle (as it stands) timed on the host: for every TT step l, one MU iteration
    on a column sample of X_l (<= budget_elems entries, real shape otherwise),
    scaled linearly in the column count, times `iters`.  Returns (seconds per full
    decomposition, threads, description)."""
    import numpy as np

    import ntt_inputs as ni
    import oracle
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    total = 0.0
    parts = []
    for l, (m, n, r) in enumerate(step_shapes(dims, ranks), start=1):
        ns = max(1, min(n, budget_elems // m))
        X = ni.uniform(m * ns, 7, 0x500 + l).reshape(m, ns)
        X = X.astype(np.float32) if l == 1 else X
        W0 = ni.uniform(m * r, 0, ni.stream_w(l)).reshape(m, r)
        H0 = ni.uniform(r * ns, 0, ni.stream_h(l)).reshape(r, ns)
        t0 = time.perf_counter()
        oracle.nmf_mu(X, W0, H0, 1)
        dt = time.perf_counter() - t0
        total += dt * (n / ns) * iters
        parts.append(f"step{l}:{m}x{ns}/{n}")
    desc = ("oracle (C, fp64, OpenMP over independent outputs) 1 MU iteration per TT step on a column sample "
            f"({', '.join(parts)}), scaled by n/sample and x{iters} iterations")
    return total, threads, desc


def run_reference(args):
    ws, rk, _ = dist_env()
    if ws > 1 and rk != 0:
        return 0
    w = workload(args.workload, args.iters)
    its = (len(w.dims) - 1) * w.iters
    times = []
    threads, desc = 1, ""
    for s in range(args.warmup + args.steps):
        t, threads, desc = oracle_sample_time(w.dims, w.ranks, w.iters)
        if s >= args.warmup:
            times.append(t)
    t = statistics.median(times)
    v = its / t
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.workload, "dims": w.dims, "ranks": w.ranks, "iters_per_step": w.iters,
                   "mu_iters_per_step": its},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "oracle", "sample": desc},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ------------------------------------------------- other BASELINE workloads ---
def other_workloads(h, P, ni, torch, steps=2):
    """nTT wall time of configs 1 and 4 and MU iterations/s of the single-NMF configs 2 and
    5 (1-GPU slice 32768 x 65536, SURVEY s.8(d) d.2) on device-generated synthetic inputs.
    Reported beside the headline workload (config 3); not part of its timed region."""
    import numpy as np
    out = {}
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    for name in ("config1", "config4", "paper256"):
        w = ni.workloads()[name]
        cores0 = torch.from_numpy(ni.make_cores(w.dims, w.ranks, w.seed).astype(np.float32)).cuda()
        A = torch.empty(w.numel, device="cuda")
        h.ntt_generate(w.dims, w.ranks, cores0, w.noise_amp, w.seed, ni.STREAM_NOISE, A)
        cores = torch.empty(P.cores_size(w.dims, w.ranks), device="cuda")
        err = h.ntt_decompose(A, w.dims, w.ranks, w.iters, w.seed, 1e-16, cores, want_error=True)
        nrep = 1 if name == "paper256" else steps
        e0, e1 = ev(), ev()
        e0.record()
        for _ in range(nrep):
            h.ntt_decompose(A, w.dims, w.ranks, w.iters, w.seed, 1e-16, cores)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / nrep
        its = (len(w.dims) - 1) * w.iters
        out[name] = {"ntt_wall_ms": ms, "mu_iter_per_s": its / (ms / 1e3), "rel_error": err,
                     "dims": w.dims, "ranks": w.ranks, "iters_per_step": w.iters,
                     "arithmetic": ARITH_NTT}
        if name == "paper256":
            out[name]["note"] = ("the paper's strong-scaling tensor (P:311-312, P:338: 256^4, TT ranks 1,10,10,10,1) "
                                 "at 1 GPU; step 1 runs k_fused_c's rank-16 class")
        del A, cores
        torch.cuda.empty_cache()
    for name, rows, iters in (("config2", None, 20), ("config5", 32768, 10)):
        w = ni.workloads()[name]
        m, n = w.dims
        r = w.ranks[0]
        if rows:
            m = rows
        dims, ranks, cores = ni.make_factor_cores(m, n, r, w.seed)
        X = torch.empty(m * n, device="cuda")
        h.ntt_generate(dims, ranks, torch.from_numpy(cores.astype(np.float32)).cuda(), w.noise_amp or 0.01, w.seed,
                       ni.STREAM_NOISE, X)
        W = torch.empty(m * r, device="cuda")
        H = torch.empty(r * n, device="cuda")
        h.ntt_fill_uniform(W, m * r, w.seed, ni.stream_w(1))
        h.ntt_fill_uniform(H, r * n, w.seed, ni.stream_h(1))
        h.ntt_nmf_mu(X, m, n, n, r, 1, 1e-16, W, H)
        e0, e1 = ev(), ev()
        e0.record()
        h.ntt_nmf_mu(X, m, n, n, r, iters, 1e-16, W, H)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        alg = 4.0 * n * (2 * m + 3 * r)  # 2-pass algorithmic bytes per iteration
        out[name] = {"mu_iter_per_s": 1e3 / ms, "ms_per_iter": ms, "m": m, "n": n, "r": r, "timed_iters": iters,
                     "effective_GBps": alg / (ms / 1e3) / 1e9,
                     "path": "tcgen05 kind::f16 fp16x2 2-pass (mu_tc16.cu)", "arithmetic": ARITH_TC,
                     "note": "config 5 on the 1-GPU row slice (SURVEY s.8(d)); inputs X = W0 H0 + noise on device"}
        # BCD NMF (Alg. 3, SURVEY s.8(f) f1) on the same X: two passes over X per iteration
        h.ntt_fill_uniform(W, m * r, w.seed, ni.stream_w(1))
        h.ntt_fill_uniform(H, r * n, w.seed, ni.stream_h(1))
        W0, H0 = W.clone(), H.clone()
        h.ntt_nmf_bcd(X, m, n, n, r, 2, W, H)
        W.copy_(W0)
        H.copy_(H0)
        e0, e1 = ev(), ev()
        e0.record()
        tr = h.ntt_nmf_bcd(X, m, n, n, r, iters, W, H, trace=True)
        e1.record()
        torch.cuda.synchronize()
        msb = e0.elapsed_time(e1) / iters
        out[name]["bcd"] = {"iter_per_s": 1e3 / msb, "ms_per_iter": msb, "timed_iters": iters,
                            "effective_GBps_2xX": 8.0 * m * n / (msb / 1e3) / 1e9,
                            "rel_error_after": float((2.0 * tr[-1]) ** 0.5 / float(torch.linalg.norm(X))),
                            "path": "ntt_nmf_bcd: one CUDA graph per iteration, fp16x2 tcgen05 X passes (bcd.cu)"}
        del X, W, H, W0, H0
        torch.cuda.empty_cache()
    # TT-SVD baseline (SURVEY s.8(f) f4) at the nTT ranks of configs 3 and 4
    for name in ("config3", "config4"):
        w = ni.workloads()[name]
        cores0 = torch.from_numpy(ni.make_cores(w.dims, w.ranks, w.seed).astype(np.float32)).cuda()
        A = torch.empty(w.numel, device="cuda")
        h.ntt_generate(w.dims, w.ranks, cores0, w.noise_amp, w.seed, ni.STREAM_NOISE, A)
        cap = P.cores_size(w.dims, [64] * (len(w.dims) - 1))
        cores = torch.empty(cap, device="cuda")
        ranks, err = h.ntt_tt_svd(A, w.dims, 0.0, cores, cap, max_ranks=w.ranks, want_error=True)
        e0, e1 = ev(), ev()
        e0.record()
        for _ in range(steps):
            h.ntt_tt_svd(A, w.dims, 0.0, cores, cap, max_ranks=w.ranks)
        e1.record()
        torch.cuda.synchronize()
        row = {"ttsvd_ms": e0.elapsed_time(e1) / steps, "ranks": ranks, "rel_error": err,
               "path": "ntt_tt_svd: fp64 Gram + one-CTA eigensolver per step (tt_svd.cu)"}
        # nTT with the paper's BCD NMF at every step (Alg. 2 + Alg. 3, SURVEY s.8(f) f1) at the same ranks
        bc = torch.empty(P.cores_size(w.dims, w.ranks), device="cuda")
        h.ntt_decompose_bcd(A, w.dims, w.ranks, w.iters, w.seed, bc)
        e0, e1 = ev(), ev()
        e0.record()
        errb = h.ntt_decompose_bcd(A, w.dims, w.ranks, w.iters, w.seed, bc, want_error=True)
        e1.record()
        torch.cuda.synchronize()
        out.setdefault(name, {})["bcd_sweep"] = {"ntt_wall_ms": e0.elapsed_time(e1), "rel_error": errb,
                                                 "iters_per_step": w.iters,
                                                 "path": "ntt_decompose_bcd: BCD NMF (Alg. 3) at every TT step"}
        del bc
        out.setdefault(name, {})["ttsvd"] = row
        del A, cores
        torch.cuda.empty_cache()
    return out


def cpu_baseline_other(other, ni, oracle_full=False):
    """The oracle timed beside the other workloads (cpu_baseline leg): the FULL config-1 nTT
    (200 MU iterations/step); the config-4 nTT, full with --oracle-full, else 3 iterations/step
    scaled to 300 (labelled extrapolated); 2 iterations of oracle.nmf_bcd on a config-2-shaped X;
    oracle.tt_svd on a config-4-shaped tensor (numpy fp64 / LAPACK; seeded inputs)."""
    import numpy as np
    import oracle
    rng = np.random.default_rng(0)
    threads = int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))
    for name in ("config1", "config4"):
        if name not in other:
            continue
        w = ni.workloads()[name]
        A = oracle.tt_full_f32(w.dims, w.ranks, ni.make_cores(w.dims, w.ranks, w.seed), w.noise_amp, w.seed)
        full = name == "config1" or oracle_full
        it = w.iters if full else 3
        t0 = time.perf_counter()
        oracle.ntt_decompose(A, w.ranks, it, seed=w.seed)
        dt = (time.perf_counter() - t0) * (w.iters / it)
        other[name]["cpu_baseline"] = {
            "value": dt * 1e3, "unit": "ms", "kind": "oracle", "cores": threads, "cpu_model": cpu_model(),
            "extrapolated": not full,
            "sample": (f"the full oracle.ntt_decompose ({w.iters} MU iterations/step)" if full else
                       f"oracle.ntt_decompose at {it} MU iterations/step, time x{w.iters // it} (extrapolated)")}
        del A
    if "config2" in other and "bcd" in other["config2"]:
        m, n, r = other["config2"]["m"], other["config2"]["n"], other["config2"]["r"]
        X = rng.random((m, n))
        t0 = time.perf_counter()
        oracle.nmf_bcd(X, rng.random((m, r)), rng.random((r, n)), 2)
        dt = (time.perf_counter() - t0) / 2
        other["config2"]["bcd"]["cpu_baseline"] = {
            "value": 1.0 / dt, "unit": "BCD-iter/s", "kind": "oracle",
            "sample": "2 iterations of oracle.nmf_bcd (numpy fp64) on a 4096 x 4096 X"}
        del X
    if "config4" in other and "ttsvd" in other["config4"]:
        w = ni.workloads()["config4"]
        A = rng.random(w.dims)
        t0 = time.perf_counter()
        oracle.tt_svd(A, 0.0, w.ranks)
        other["config4"]["ttsvd"]["cpu_baseline"] = {
            "value": (time.perf_counter() - t0) * 1e3, "unit": "ms", "kind": "oracle",
            "sample": "one oracle.tt_svd (LAPACK SVD per step, fp64) of a 6^10 tensor at ranks 5"}
        del A


# ------------------------------------------------------------------- ours ---
def run_ours(args):
    import numpy as np
    import torch

    import ntt_inputs as ni
    import paper_2008_01340_b200 as P

    ws, rk, lr = dist_env()
    torch.cuda.set_device(lr)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", lr))
    w = workload(args.workload, args.iters)
    dims, ranks, iters = list(w.dims), list(w.ranks), w.iters
    d = len(dims)
    its = (d - 1) * iters
    stream = torch.cuda.current_stream()
    if ws > 1:
        uid = [P.ntt_get_unique_id() if rk == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        h = P.Handle(lr, stream.cuda_stream, unique_id=uid[0], nranks=ws, rank=rk)
    else:
        h = P.Handle(lr, stream.cuda_stream)

    # synthetic input: random TT cores, contracted + noise on device
    cores0 = ni.make_cores(dims, ranks, w.seed)
    b, off = P.ntt_dist_block(dims[-1], ws, rk)
    ldims = dims[:-1] + [b]
    fr = [1, *ranks, 1]
    last = cores0[-fr[d - 1] * dims[-1]:].reshape(fr[d - 1], dims[-1])[:, off:off + b]
    lcores = np.concatenate([cores0[:-fr[d - 1] * dims[-1]], last.ravel()]).astype(np.float32)
    Nloc = int(np.prod(ldims))
    A = torch.empty(Nloc, dtype=torch.float32, device="cuda")
    h.ntt_generate(ldims, ranks, torch.from_numpy(lcores).cuda(), w.noise_amp, w.seed, ni.STREAM_NOISE, A)
    cores = torch.empty(P.cores_size(dims, ranks), dtype=torch.float32, device="cuda")

    def step():
        return h.ntt_decompose(A, dims, ranks, iters, w.seed, 1e-16, cores, want_error=True)

    for _ in range(args.warmup):
        err = step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = ClockSampler(lr)
    clk.start()
    l0 = h.launch_count
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        err = step()
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = clk.stop()
    launches = h.launch_count - l0
    ms = e0.elapsed_time(e1) / args.steps
    # per-kernel-class profile in a SEPARATE run (the profiler's events and per-call fold are
    # not in the timed region above): re-capture with profiling on, one untimed step, then K
    h.ntt_profile_enable(True)
    step()
    h.ntt_profile_enable(True)  # reset the counters; the graph (captured with profiling) is kept
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for _ in range(args.steps):
        step()
    p1.record(stream)
    torch.cuda.synchronize()
    prof_ms = p0.elapsed_time(p1) / args.steps
    step_prof = {(c, l): h.ntt_profile_get(c, l) for c in range(8) for l in range(0, d + 1)}
    h.ntt_profile_enable(False)
    # read-only HBM stream ceiling over the input buffer
    ceiling = h.ntt_stream_ceiling(A, (A.numel() * 4) // 16 * 16, 5)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    # ---- e2e: same call with HOST buffers (pinned), H2D/D2H inside the call
    e2e = None
    if not args.no_e2e:
        Ah = torch.empty(Nloc, dtype=torch.float32, pin_memory=True)
        Ah.copy_(A)
        ch = torch.empty(cores.numel(), dtype=torch.float32, pin_memory=True)
        h.ntt_decompose(Ah, dims, ranks, iters, w.seed, 1e-16, ch, want_error=True)  # warm staging buffers
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for _ in range(args.steps):
            h.ntt_decompose(Ah, dims, ranks, iters, w.seed, 1e-16, ch, want_error=True)
        q1.record(stream)
        torch.cuda.synchronize()
        ems = q0.elapsed_time(q1) / args.steps
        if dist:
            t = torch.tensor([ems], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        # the same steps as a stream of inputs: step k+1's H2D (ntt_prefetch_input, pinned host
        # memory -> the next of two device slots, on the library's copy stream) overlaps step k's
        # decomposition; every step still copies its 4.29 GB and reads its cores + error back.
        # Wall clock around all K steps, synchronised on both sides (first copy not overlapped).
        h.ntt_prefetch_input(Ah, Nloc)
        h.ntt_decompose(Ah, dims, ranks, iters, w.seed, 1e-16, ch, want_error=True)  # warm slots + graphs
        h.ntt_prefetch_input(Ah, Nloc)
        h.ntt_decompose(Ah, dims, ranks, iters, w.seed, 1e-16, ch, want_error=True)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        tp0 = time.perf_counter()
        h.ntt_prefetch_input(Ah, Nloc)
        for k in range(args.steps):
            if k + 1 < args.steps:
                h.ntt_prefetch_input(Ah, Nloc)
            h.ntt_decompose(Ah, dims, ranks, iters, w.seed, 1e-16, ch, want_error=True)
        torch.cuda.synchronize()
        pms = (time.perf_counter() - tp0) * 1e3 / args.steps
        if dist:
            t = torch.tensor([pms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            pms = float(t.item())
        e2e = {"value": its / (pms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(Nloc * 4) * ws,
               "d2h_bytes_per_step": int(cores.numel() * 4 + 8) * ws, "ms_per_step": pms,
               "pipelined": ("step k+1's host-to-device copy (ntt_prefetch_input, pinned memory, the library's "
                             "copy stream, two device input slots) overlaps step k's decomposition; wall clock "
                             "over all steps, the first copy not overlapped"),
               "serial_ms_per_step": ems, "serial_value": its / (ems / 1e3)}
        del Ah

    # ---- roofline: dominant kernel = the fused 1-pass X-stream kernel on TT step 1
    #      (k_fused<8,4>: S = W^T X, H update, next X H^T / H H^T), class 0 step 1
    pk, pk_kind = peaks()
    n0, ms0, by0 = step_prof[(0, 1)]
    achieved = (by0 / (ms0 / 1e3)) / 1e9 if ms0 > 0 else 0.0
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            traffic = json.load(f).get(args.workload, {}).get("dram_bytes_per_launch")
    except Exception:
        pass
    per_step = {}
    for l in range(1, d + 1):
        ent = {}
        for c, nm in enumerate(["xstream", "xht", "wupdate", "ttstream", "other", "hpass2", "tc_xht", "tc_wtx"]):
            k, t, by = step_prof[(c, l)]
            if k:
                ent[nm] = {"launches_per_step": k // args.steps, "ms_per_step": t / args.steps,
                           "GBps": (by / (t / 1e3)) / 1e9 if t > 0 else None}
        per_step[f"step{l}" if l < d else "last_core+error"] = ent
    roofline = {"bound": "hbm", "achieved": achieved, "peak": pk, "unit": "GB/s", "frac": achieved / pk,
                "traffic": traffic, "peak_kind": pk_kind,
                "kernel": "k_fused_m (persistent 1-pass MU launch of TT step 1 on mma.sync with the X16 cache: "
                          "32 x 33554432, r=8; prologue + 100 passes)",
                "launches": n0, "kernel_ms_per_step": ms0 / args.steps,
                "kernel_share_of_step": (ms0 / args.steps) / prof_ms if prof_ms > 0 else None,
                "profiled_ms_per_step": prof_ms,
                "algorithmic_bytes_per_launch": by0 / n0 if n0 else None,
                "frac_of": {"measured_copy_peak": achieved / pk, "8TBs_nominal": achieved / 8000.0,
                            "read_stream_ceiling": achieved / ceiling if ceiling > 0 else None},
                "read_stream_ceiling_GBps": ceiling,
                "pct_of_8TBs": achieved / 8000.0, "per_tt_step": per_step}

    line = {
        "metric": METRIC, "value": its / (ms / 1e3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if ws > 1 else "strong",
        "vs_baseline": None, "dtype": "f32", "arithmetic": ARITH_NTT, "data": "synthetic",
        "config": {"workload": args.workload, "dims": dims, "ranks": ranks, "iters_per_step": iters,
                   "mu_iters_per_step": its, "noise": f"{w.noise} amp {w.noise_amp}",
                   "l2": "input (4.29 GB) larger than L2; no flush", "parallelism": f"last-mode x{ws}",
                   "ntt_wall_ms": ms, "rel_error": err},
        "roofline": roofline,
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": e2e,
    }
    if ws == 1 and not args.no_other:
        line["other_workloads"] = other_workloads(h, P, ni, torch)
    if rk == 0 and ws == 1 and not args.no_cpu:
        t, threads, desc = oracle_sample_time(dims, ranks, iters)
        line["cpu_baseline"] = {"value": its / t, "unit": UNIT, "cores": threads, "cpu_model": cpu_model(),
                                "kind": "oracle", "sample": desc, "extrapolated": True}
        if "other_workloads" in line:
            cpu_baseline_other(line["other_workloads"], ni, args.oracle_full)
    if rk == 0:
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
