"""Seeded synthetic-input generators shared by the tests, the bench and smoke().

This module holds NONE of the method's arithmetic (no MU step, no contraction,
no error metric).  It provides:

* the counter-based RNG spec, vectorised in numpy --
  u(seed, stream, i) = (mix64(mix64(seed ^ mix64(stream + G)) + (i+1) G) >> 40) * 2^-24,
  mix64 = the SplitMix64 finaliser, G = 0x9E3779B97F4A7C15.  The oracle (C) and
  the CUDA path implement the same text independently; tests pin all three to
  each other bit for bit;
* random TT cores ("each of the tensor train factors ... sampled from
  a uniform distribution between 0 and 1") and noise draws;
* the five BASELINE.json workload recipes (shapes, ranks, iterations, noise).

Building the tensor itself from the cores is Eq. 1 -- that is the oracle's job
in the tests (``oracle.tt_full_f32``) and the product's job in the bench
(``ntt_generate``); it is deliberately not here.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)

# RNG stream ids (reading R20)
STREAM_CORE_BASE = 0x100   # core l of a generated train: 0x100 + l (l = 1..d)
STREAM_NOISE = 0x300       # additive uniform noise
STREAM_BM1 = 0x301         # Box-Muller u1
STREAM_BM2 = 0x302         # Box-Muller u2
STREAM_W0 = 0x400          # ground-truth W0 (configs 2, 5)
STREAM_H0 = 0x401          # ground-truth H0 (configs 2, 5)


def stream_w(l: int) -> int:
    return 0x200 + 2 * l


def stream_h(l: int) -> int:
    return 0x201 + 2 * l


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def rng_u24(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Top-24-bit integer draws for the given global indices (uint32)."""
    with np.errstate(over="ignore"):
        s = np.array([seed], dtype=np.uint64)
        st = np.array([stream], dtype=np.uint64)
        key = _mix64(s ^ _mix64(st + GOLDEN))[0]
        i = np.asarray(idx, dtype=np.uint64)
        v = _mix64(key + (i + np.uint64(1)) * GOLDEN)
    return (v >> np.uint64(40)).astype(np.uint32)


def uniform(count: int, seed: int, stream: int, offset: int = 0, dtype=np.float64,
            chunk: int = 1 << 24) -> np.ndarray:
    """u(seed, stream, offset + i) for i < count; values k*2^-24 in [0, 1)."""
    out = np.empty(count, dtype=dtype)
    for a in range(0, count, chunk):
        b = min(count, a + chunk)
        idx = np.arange(offset + a, offset + b, dtype=np.uint64)
        out[a:b] = rng_u24(seed, stream, idx).astype(np.float64) * (1.0 / 16777216.0)
    return out


def abs_normal(count: int, seed: int, offset: int = 0) -> np.ndarray:
    """|z|, z ~ N(0,1) by Box-Muller from streams 0x301/0x302 (fp64):
    z = sqrt(-2 ln(1 - u1)) cos(2 pi u2)."""
    u1 = uniform(count, seed, STREAM_BM1, offset)
    u2 = uniform(count, seed, STREAM_BM2, offset)
    return np.abs(np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2))


def full_ranks(ranks) -> List[int]:
    return [1, *[int(r) for r in ranks], 1]


def cores_size(dims, ranks) -> int:
    fr = full_ranks(ranks)
    return int(sum(fr[l] * dims[l] * fr[l + 1] for l in range(len(dims))))


def make_cores(dims, ranks, seed: int = 0, streams: Optional[List[int]] = None) -> np.ndarray:
    """Packed random TT cores, core l (1-based) of shape (r_{l-1}, n_l, r_l) row-major,
    entries u(seed, 0x100 + l, flat index within the core)."""
    fr = full_ranks(ranks)
    parts = []
    for l in range(1, len(dims) + 1):
        sz = fr[l - 1] * dims[l - 1] * fr[l]
        st = streams[l - 1] if streams is not None else STREAM_CORE_BASE + l
        parts.append(uniform(sz, seed, st))
    return np.concatenate(parts)


def make_cores_decay(dims, ranks, rho: float, seed: int = 0) -> np.ndarray:
    """Packed non-negative TT cores with a graded spectrum (the eps-sweep input of SURVEY s.8(f)
    f2): the entries of make_cores scaled by rho^(a + b), a / b the left / right bond index of the
    entry, so that bond direction k carries ~rho^k of the energy and the unfoldings' singular
    values decay geometrically instead of the U[0,1) train's one dominant direction plus a flat
    rest.  rho in (0, 1]; rho = 1 gives make_cores."""
    c = make_cores(dims, ranks, seed)
    fr = full_ranks(ranks)
    out = np.empty_like(c)
    o = 0
    for l in range(len(dims)):
        a, n, b = fr[l], dims[l], fr[l + 1]
        s = np.power(float(rho), np.add.outer(np.arange(a), np.arange(b)))
        out[o:o + a * n * b] = (c[o:o + a * n * b].reshape(a, n, b) * s[:, None, :]).ravel()
        o += a * n * b
    return out


def make_factor_cores(m: int, n: int, r: int, seed: int = 0) -> Tuple[List[int], List[int], np.ndarray]:
    """X = W0 H0 written as a d=2 train (W0: 1 x m x r, H0: r x n x 1) with W0, H0 drawn
    from streams 0x400 / 0x401 (configs 2 and 5)."""
    cores = make_cores([m, n], [r], seed, streams=[STREAM_W0, STREAM_H0])
    return [m, n], [r], cores


@dataclass
class Workload:
    name: str
    kind: str                      # "ntt" (tensor-train sweep) or "nmf" (single NMF)
    dims: List[int]
    ranks: List[int]               # inner TT ranks (ntt) or [r] for nmf
    iters: int
    noise: str = "none"            # "none" | "uniform" | "absnormal"
    noise_amp: float = 0.0
    seed: int = 0
    note: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def numel(self) -> int:
        return int(np.prod(self.dims))


def workloads() -> dict:
    """BASELINE.json configs 1..5 (noise readings R12)."""
    return {
        "config1": Workload("config1", "ntt", [5, 4, 5, 6], [4, 3, 2], 200,
                            note="Fig. 1 shape (P:62), exact TT, cores U[0,1) seed 0"),
        "config2": Workload("config2", "nmf", [4096, 4096], [16], 500, noise="absnormal", noise_amp=0.01,
                            note="X = W0 H0 + 0.01|N(0,1)|, W0/H0 U[0,1) rank 16"),
        "config3": Workload("config3", "ntt", [32] * 6, [8] * 5, 100, noise="uniform", noise_amp=5.12,
                            note="32^6 TT ranks 8 + 1% uniform noise (0.01 * mean 512 * u)"),
        "config4": Workload("config4", "ntt", [6] * 10, [5] * 9, 300,
                            note="6^10 exact TT ranks 5"),
        "config5": Workload("config5", "nmf", [131072, 65536], [32], 100, noise="uniform", noise_amp=0.08,
                            note="X = W0 H0 + 0.08 u (1% of mean 8); 1-GPU slice 32768 rows",
                            extra={"slice_rows": 32768}),
        # SURVEY s.8(f) f3: the paper's strong-scaling tensor shape, synthetic
        "paper256": Workload("paper256", "ntt", [256] * 4, [10, 10, 10], 100, noise="uniform", noise_amp=0.625,
                             note="256^4 (16 GiB) TT ranks 10 + 1% uniform noise (0.01 * mean 62.5 * u)"),
    }


def bcd_overshoot_matrix(m: int, n: int, r: int, seed: int, kind: str = "colscaled", extra: int = 1) -> np.ndarray:
    """A non-negative m x n test matrix on which Alg. 3's extrapolation overshoots by itself
    (the l.17 correction fires twice or more within 100 iterations for the seeds the tests
    use): a rank-(r + extra) non-negative product -- so a rank-r fit keeps a residual well
    above the fp32 resolution of the objective -- with row ("scaled") or column ("colscaled")
    scales spread over three decades, rounded to fp32.  numpy's default_rng(seed); no method
    arithmetic."""
    rng = np.random.default_rng(seed)
    base = rng.random((m, r + extra)) @ rng.random((r + extra, n))
    if kind == "scaled":
        X = (10.0 ** rng.uniform(-1.5, 1.5, (m, 1))) * base
    else:
        X = base * (10.0 ** rng.uniform(-1.5, 1.5, (1, n)))
    return X.astype(np.float32)
