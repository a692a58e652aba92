"""paper_2008_01340_b200 -- B200-native MU-NMF non-negative tensor train.

Thin Python binding of libntt.so (include/ntt.h), arXiv 2008.01340.  Functions
keep the C names (``ntt_nmf_mu``, ``ntt_decompose``, ``ntt_reconstruct`` ...)
and accept torch tensors (CUDA or CPU) or raw integer pointers; they only
marshal arguments -- every step of the hot path runs in the library's sm_100a
kernels.  PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

from ._lib import LIB_PATH, lib  # noqa: F401

__all__ = [
    "NttError", "Handle", "ntt_compression_ratio", "ntt_decompose_workspace_bytes", "ntt_dist_block",
    "ntt_get_unique_id", "STREAM_NOISE", "stream_w", "stream_h", "cores_size", "LIB_PATH",
]

STREAM_NOISE = 0x300


def stream_w(l: int) -> int:
    return 0x200 + 2 * l


def stream_h(l: int) -> int:
    return 0x201 + 2 * l


class NttError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"ntt status {status}: {msg}")
        self.status = status


def _ptr(x) -> Optional[int]:
    """Pointer of a torch tensor / numpy array / int / None (no copies made)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return x.ctypes.data
    raise TypeError(f"cannot take a pointer of {type(x)}")


def _i64arr(v: Sequence[int]):
    return (ctypes.c_int64 * len(v))(*[int(x) for x in v])


def _i32arr(v: Sequence[int]):
    return (ctypes.c_int32 * max(1, len(v)))(*[int(x) for x in v])


def cores_size(dims, ranks) -> int:
    fr = [1, *ranks, 1]
    return int(sum(fr[l] * dims[l] * fr[l + 1] for l in range(len(dims))))


def ntt_compression_ratio(dims, ranks) -> float:
    return float(lib().ntt_compression_ratio(len(dims), _i64arr(dims), _i32arr(ranks)))


def ntt_decompose_workspace_bytes(dims, ranks) -> int:
    return int(lib().ntt_decompose_workspace_bytes(len(dims), _i64arr(dims), _i32arr(ranks)))


def ntt_dist_block(n_last: int, nranks: int, rank: int):
    off = ctypes.c_int64(0)
    b = lib().ntt_dist_block(n_last, nranks, rank, ctypes.byref(off))
    return int(b), int(off.value)


def ntt_get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    st = lib().ntt_get_unique_id(buf)
    if st != 0:
        raise NttError(st, "ntt_get_unique_id failed")
    return buf.raw


class Handle:
    """Owns an ntt_handle bound to (device, stream)."""

    def __init__(self, device: int = 0, stream: Optional[int] = None, unique_id: Optional[bytes] = None,
                 nranks: int = 1, rank: int = 0, grid: Optional[tuple] = None):
        self._h = ctypes.c_void_p()
        if stream is None:
            try:
                import torch
                stream = torch.cuda.current_stream(device).cuda_stream
            except Exception:
                stream = 0
        if unique_id is None:
            st = lib().ntt_create(ctypes.byref(self._h), device, ctypes.c_void_p(stream))
        else:
            idb = ctypes.create_string_buffer(unique_id, 128)
            pr, pc = grid if grid is not None else (1, nranks)
            st = lib().ntt_create_dist_grid(ctypes.byref(self._h), device, ctypes.c_void_p(stream), idb, nranks, rank,
                                            pr, pc)
        if st != 0:
            raise NttError(st, f"ntt_create failed ({lib().ntt_status_string(st).decode()})")

    # -------------------------------------------------------------- plumbing
    def _check(self, st: int):
        if st != 0:
            raise NttError(st, f"{lib().ntt_status_string(st).decode()}: {lib().ntt_last_error(self._h).decode()}")

    def close(self):
        if self._h:
            lib().ntt_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream: int):
        self._check(lib().ntt_set_stream(self._h, ctypes.c_void_p(stream)))

    @property
    def launch_count(self) -> int:
        return int(lib().ntt_launch_count(self._h))

    @property
    def rank(self) -> int:
        return int(lib().ntt_dist_rank(self._h))

    @property
    def size(self) -> int:
        return int(lib().ntt_dist_size(self._h))

    @property
    def grid(self):
        """(pr, pc, ga, gb): process-grid shape and this rank's (row, column) position."""
        v = [ctypes.c_int() for _ in range(4)]
        lib().ntt_dist_grid(self._h, *[ctypes.byref(x) for x in v])
        return tuple(int(x.value) for x in v)

    def last_error(self) -> str:
        return lib().ntt_last_error(self._h).decode()

    # ------------------------------------------------------------------ ABI
    def ntt_fill_uniform(self, p, count: int, seed: int, stream: int, index_offset: int = 0):
        self._check(lib().ntt_fill_uniform(self._h, _ptr(p), count, seed, stream, index_offset))

    def ntt_nmf_mu(self, X, m: int, n: int, ldx: int, r: int, iters: int, eps: float, W, H, trace: bool = False):
        tr = (ctypes.c_double * max(1, iters))() if trace else None
        self._check(lib().ntt_nmf_mu(self._h, _ptr(X), m, n, ldx, r, iters, eps, _ptr(W), _ptr(H), tr))
        return list(tr)[:iters] if trace else None

    def ntt_prefetch_input(self, A, count: int):
        """Asynchronous H2D copy of a host tensor into the handle's next input slot (ntt_prefetch_input)."""
        self._check(lib().ntt_prefetch_input(self._h, _ptr(A), count))

    def mu_path(self, m: int, n: int, r: int) -> int:
        """ntt_debug_mu_path: 1 tiny, 2 cluster, 3 persistent 1-pass, 4 per-pass 1-pass, 5 tc, 6 generic."""
        return int(lib().ntt_debug_mu_path(self._h, m, n, r))

    def ntt_stream_ceiling(self, buf, nbytes: int, reps: int = 10) -> float:
        """Read-only HBM stream rate over a device buffer in GB/s (BASELINE.md s.3 ceiling)."""
        g = ctypes.c_double(0.0)
        self._check(lib().ntt_stream_ceiling(self._h, _ptr(buf), nbytes, reps, ctypes.byref(g)))
        return float(g.value)

    def ntt_set_dist_exchange(self, mode: int):
        """1: in-kernel NVLink exchange of the pass partials (default); 0: per-pass ncclAllReduce."""
        self._check(lib().ntt_set_dist_exchange(self._h, int(mode)))

    @property
    def peer_exchange_count(self) -> int:
        return int(lib().ntt_peer_exchange_count(self._h))

    @property
    def collective_count(self) -> int:
        return int(lib().ntt_collective_count(self._h))

    def ntt_debug_fill_uniform_cols(self, H, r: int, nloc: int, b: int, nd: int, off: int, nglob: int,
                                    seed: int, stream: int):
        self._check(lib().ntt_debug_fill_uniform_cols(self._h, _ptr(H), r, nloc, b, nd, off, nglob, seed, stream))

    def ntt_debug_gather_last_core(self, gath, r: int, nd: int, nranks: int, core):
        self._check(lib().ntt_debug_gather_last_core(self._h, _ptr(gath), r, nd, nranks, _ptr(core)))

    def ntt_set_validation(self, nonneg: bool = True):
        """NTT_VALIDATE_NONNEG: check X / A for negative or NaN entries before each call."""
        self._check(lib().ntt_set_validation(self._h, 1 if nonneg else 0))

    def ntt_debug_bcd_force_correct(self, iterations=()):
        """Test hook: the BCD iterations listed (0-based, < 52) take the correction branch."""
        mask = 0
        for i in iterations:
            mask |= 1 << int(i)
        self._check(lib().ntt_debug_bcd_force_correct(self._h, mask))

    def ntt_nmf_bcd(self, X, m: int, n: int, ldx: int, r: int, iters: int, W, H, delta: float = 0.9999,
                    trace: bool = False):
        """Alg. 3 BCD NMF on device buffers (W, H in/out); returns the accepted-objective trace if asked."""
        tr = (ctypes.c_double * max(1, iters))() if trace else None
        self._check(lib().ntt_nmf_bcd(self._h, _ptr(X), m, n, ldx, r, iters, delta, _ptr(W), _ptr(H), tr))
        return list(tr)[:iters] if trace else None

    def ntt_decompose(self, A, dims, ranks, iters: int, seed: int, eps: float, cores, workspace=None,
                      workspace_bytes: int = 0, want_error: bool = False) -> Optional[float]:
        err = ctypes.c_double(-1.0) if want_error else None
        self._check(lib().ntt_decompose(self._h, _ptr(A), len(dims), _i64arr(dims), _i32arr(ranks), iters, seed, eps,
                                        _ptr(cores), ctypes.byref(err) if err is not None else None,
                                        _ptr(workspace), workspace_bytes))
        return float(err.value) if want_error else None

    def ntt_profile_enable(self, enable: bool = True):
        self._check(lib().ntt_profile_enable(self._h, 1 if enable else 0))

    def ntt_profile_get(self, cls: int, step: int = -1):
        """(launches, total_ms, total_algorithmic_bytes) for kernel class `cls` (optionally one TT step)."""
        n, ms, by = ctypes.c_int64(0), ctypes.c_double(0), ctypes.c_double(0)
        self._check(lib().ntt_profile_get_step(self._h, cls, step, ctypes.byref(n), ctypes.byref(ms),
                                               ctypes.byref(by)))
        return int(n.value), float(ms.value), float(by.value)

    def ntt_reconstruct(self, dims, ranks, cores, out=None, ref=None, want_error: bool = False) -> Optional[float]:
        err = ctypes.c_double(-1.0) if want_error else None
        self._check(lib().ntt_reconstruct(self._h, len(dims), _i64arr(dims), _i32arr(ranks), _ptr(cores), _ptr(out),
                                          _ptr(ref), ctypes.byref(err) if err is not None else None))
        return float(err.value) if want_error else None

    def ntt_decompose_eps(self, A, dims, tt_eps: float, iters: int, seed: int, eps: float, cores,
                          cores_capacity: int, max_ranks=None, want_error: bool = False):
        """Alg. 2 with the SVD rank rule (l.5-6); returns (ranks, rel_err or None)."""
        d = len(dims)
        rk = (ctypes.c_int32 * max(d - 1, 1))()
        err = ctypes.c_double(-1.0) if want_error else None
        mr = _i32arr(max_ranks) if max_ranks is not None else None
        self._check(lib().ntt_decompose_eps(self._h, _ptr(A), d, _i64arr(dims), tt_eps, mr, iters, seed, eps,
                                            _ptr(cores), cores_capacity, rk,
                                            ctypes.byref(err) if err is not None else None))
        return [int(x) for x in rk][: d - 1], (float(err.value) if want_error else None)

    def ntt_decompose_bcd(self, A, dims, ranks, iters: int, seed: int, cores, delta: float = 0.9999,
                          want_error: bool = False) -> Optional[float]:
        """Alg. 2 with the BCD NMF (Alg. 3) at every step; returns rel_err if asked."""
        err = ctypes.c_double(-1.0) if want_error else None
        self._check(lib().ntt_decompose_bcd(self._h, _ptr(A), len(dims), _i64arr(dims), _i32arr(ranks), iters, seed,
                                            delta, _ptr(cores), ctypes.byref(err) if err is not None else None))
        return float(err.value) if want_error else None

    def ntt_tt_svd(self, A, dims, tt_eps: float, cores, cores_capacity: int, max_ranks=None,
                   want_error: bool = False):
        """TT-SVD baseline (f4) with the rank rule; returns (ranks, rel_err or None)."""
        d = len(dims)
        rk = (ctypes.c_int32 * max(d - 1, 1))()
        err = ctypes.c_double(-1.0) if want_error else None
        mr = _i32arr(max_ranks) if max_ranks is not None else None
        self._check(lib().ntt_tt_svd(self._h, _ptr(A), d, _i64arr(dims), tt_eps, mr, _ptr(cores), cores_capacity, rk,
                                     ctypes.byref(err) if err is not None else None))
        return [int(x) for x in rk][: d - 1], (float(err.value) if want_error else None)

    def ntt_rank_rule(self, X, m: int, n: int, ldx: int, tt_eps: float, want_eig: bool = False):
        """SVD rank rule on a device matrix; returns (rank, eigenvalues ascending or None)."""
        r = ctypes.c_int32()
        eig = (ctypes.c_double * min(m, n))() if want_eig else None
        self._check(lib().ntt_rank_rule(self._h, _ptr(X), m, n, ldx, tt_eps, ctypes.byref(r), eig))
        return int(r.value), (list(eig) if want_eig else None)

    def ntt_generate(self, dims, ranks, cores, noise_amp: float, seed: int, noise_stream: int, out):
        self._check(lib().ntt_generate(self._h, len(dims), _i64arr(dims), _i32arr(ranks), _ptr(cores), noise_amp,
                                       seed, noise_stream, _ptr(out)))
