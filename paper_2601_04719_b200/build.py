"""Build libkvq.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2601_04719_b200.build [--verbose]

No JIT cache, no torch extension machinery: one shared library with a plain
C ABI (include/kvq.h) that travels with the repo to the GPU box.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libkvq.so")
SOURCES = ["api.cu", "quant_kernels.cu", "metrics_kernels.cu", "attn_tc.cu", "fp8_kernels.cu", "lowbit_kernels.cu", "append_kernels.cu", "scores_codes.cu", "step_small.cu", "synth.cu", "peer.cu", "comm.cpp"]
HEADERS = ["kvq_internal.h", "device_common.cuh", "tc_common.cuh", "rt64.cuh"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# IEEE arithmetic everywhere (bit-exact parity needs it): no fast-math, no FTZ,
# IEEE division/sqrt.  Products that must not be contracted use __fmul_rn etc.
NVFLAGS = ["-O3", "-lineinfo", "-std=c++17", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
           "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    return "nvcc"


def nccl_include() -> str:
    site = sysconfig.get_paths()["purelib"]
    p = os.path.join(site, "nvidia", "nccl", "include")
    if os.path.exists(os.path.join(p, "nccl.h")):
        return p
    for p in ("/usr/include", "/usr/local/include"):
        if os.path.exists(os.path.join(p, "nccl.h")):
            return p
    raise RuntimeError("nccl.h not found (pip nvidia-nccl wheel or system NCCL headers)")


def _inputs():
    files = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    files += [os.path.join(ROOT, "include", h) for h in ("kvq.h", "kvq_synth.h")]
    files.append(os.path.abspath(__file__))
    return files


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in _inputs())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    objdir = os.path.join(PKG, "build")
    os.makedirs(objdir, exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", nccl_include()]
    objs = []
    for s in SOURCES:
        o = os.path.join(objdir, s.rsplit(".", 1)[0] + ".o")
        extra = os.environ.get("KVQ_NVCC_EXTRA", "").split()  # experiments only (e.g. -DKVQ_SPIN_ALL)
        cmd = [nvcc(), *ARCH, *NVFLAGS, *extra, *inc, "-c", os.path.join(CSRC, s), "-o", o]
        if verbose and s.endswith(".cu"):
            cmd += ["-Xptxas", "-v"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        objs.append(o)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv))
