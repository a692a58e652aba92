"""CPU-side checks of the C ABI: the library loads and exports every symbol
include/ntt.h declares; host-only entry points behave (no GPU compute here)."""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2008_01340_b200 as P
from paper_2008_01340_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    txt = open(os.path.join(ROOT, "include", "ntt.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ntt_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = _declared()
    assert len(names) >= 15
    for nm in names:
        assert hasattr(L, nm), nm
    # the binding covers the whole ABI, with the same names
    assert set(names) == set(_lib.SIGNATURES)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for nm in names:
        assert re.search(rf"\bT {nm}\b", out), nm


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(80|86|89|90)", out)


def test_library_does_not_link_the_oracle():
    out = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "ora_" not in out
    deps = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in deps


def test_host_only_entry_points(ora):
    assert _lib.lib().ntt_abi_version() == 1
    for dims, ranks in [([5, 4, 5, 6], [4, 3, 2]), ([32] * 6, [8] * 5), ([6] * 10, [5] * 9), ([2, 2, 2, 2], [1, 1, 1])]:
        assert P.ntt_compression_ratio(dims, ranks) == pytest.approx(ora.compression_ratio(dims, ranks), rel=1e-15)
        assert P.ntt_decompose_workspace_bytes(dims, ranks) > 0
    assert P.ntt_decompose_workspace_bytes([5, 4], [9]) == 0  # invalid rank -> 0
    assert P.ntt_compression_ratio([5, 0], [1]) < 0
    assert _lib.lib().ntt_status_string(3) == b"rank error"


@pytest.mark.parametrize("n,p", [(32, 8), (6, 4), (7, 3), (1, 1), (100, 7)])
def test_dist_block_partition(n, p):
    blocks = [P.ntt_dist_block(n, p, g) for g in range(p)]
    off = 0
    for b, o in blocks:
        assert o == off and b >= 0
        off += b
    assert off == n
    sizes = [b for b, _ in blocks]
    assert max(sizes) - min(sizes) <= 1
    assert P.ntt_dist_block(n, p, p)[0] == -1


def test_handle_creation_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    with pytest.raises(P.NttError):
        P.Handle(0, stream=0)
