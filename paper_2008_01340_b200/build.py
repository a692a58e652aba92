"""Build libntt.so (the product's CUDA library) in-tree with nvcc for sm_100a.

    python -m paper_2008_01340_b200.build        # or __graft_entry__.build()
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# experiment builds: NTT_NVCC_DEFS="-DFOO=1" NTT_LIB_OUT=/path/libntt_x.so (own object dir)
_VARIANT = os.environ.get("NTT_LIB_OUT")
OBJ = os.path.join(PKG, "build_obj" + ("_" + os.path.basename(_VARIANT).replace(".so", "") if _VARIANT else ""))
LIB = _VARIANT or os.path.join(PKG, "libntt.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    return p


def nccl_include() -> str:
    cands = [os.path.join(sysconfig.get_paths()["purelib"], "nvidia", "nccl", "include"), "/usr/include"]
    for c in cands:
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found (needed for types only; NCCL itself is dlopen'ed)")


def flags():
    extra = ["-DNTT_WATCHDOG"] if os.environ.get("NTT_WATCHDOG") else []
    extra += os.environ.get("NTT_NVCC_DEFS", "").split()
    return [*extra, "-O3", "-lineinfo", "-std=c++17", *ARCH, "-Xcompiler", "-fPIC,-O3", "-Xptxas", "-v",
            f"-I{os.path.join(ROOT, 'include')}", f"-I{nccl_include()}", "--expt-relaxed-constexpr"]


def _compile(src: str) -> str:
    os.makedirs(OBJ, exist_ok=True)
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    deps = glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "ntt.h"), src]
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(d) for d in deps):
        return obj
    cmd = [nvcc(), *flags(), "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
    with open(obj + ".ptxas.log", "w") as f:
        f.write(res.stderr)
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if force and os.path.isdir(OBJ):
        shutil.rmtree(OBJ)
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        objs = list(ex.map(_compile, srcs))
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc(), *ARCH, "-shared", "-o", LIB, *objs, "-ldl"]
        subprocess.check_call(cmd)
    if verbose:
        print(LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
