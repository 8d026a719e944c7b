"""Build librlpolicy.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2605_15565_b200.build [--force] [-v]

Every .cu under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` (advantage.cu additionally with
``-fmad=false``: its fp64 arithmetic must not be FMA-contracted, reading Z7) and
linked against the NCCL 2.28 that ships with torch (same libnccl.so.2 torch loads).
ptxas resource usage (-Xptxas -v) is written to build/ptxas.log.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "librlpolicy.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    cands = []
    try:
        import nvidia.nccl as _n  # torch's bundled NCCL
        base = list(_n.__path__)[0]
        cands.append(base)
    except Exception:
        pass
    cands.append("/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl")
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return os.path.join(c, "include"), os.path.join(c, "lib")
    raise RuntimeError("nccl.h not found (expected torch's nvidia/nccl package)")


def _nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale(force: bool) -> bool:
    if force or not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "rl_policy.h"), os.path.abspath(__file__)]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, variant: str = "") -> str:
    """variant "trace": a development build with -DRL_VC_TRACE (vp_cache_kernel cycle counters,
    rl_debug_vc_trace) into librlpolicy_trace.so; variant "checks": -DRL_DEBUG_CHECKS (device-side
    bounds assertions) into librlpolicy_checks.so.  Neither is the product library."""
    global BUILD, LIB
    if variant:
        BUILD = os.path.join(ROOT, f"build_{variant}")
        LIB = os.path.join(PKG, f"librlpolicy_{variant}.so")
    if not _stale(force):
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    nccl_inc, nccl_lib = _nccl_dirs()
    nvcc = _nvcc()
    common = [nvcc, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
              "-I", os.path.join(ROOT, "include"), "-I", nccl_inc, "-Xptxas", "-v",
              "--expt-relaxed-constexpr"] + {"trace": ["-DRL_VC_TRACE"], "checks": ["-DRL_DEBUG_CHECKS"],
                                           "ab": ["-DRL_AB"]}.get(variant, [])
    def compile_one(src):
        obj = os.path.join(BUILD, os.path.basename(src).replace(".cu", ".o"))
        extra = ["-fmad=false"] if os.path.basename(src) == "advantage.cu" else []
        cmd = common + extra + ["-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        return src, obj, subprocess.run(cmd, capture_output=True, text=True)

    objs, logs = [], []
    # one nvcc per translation unit, in parallel (the tcgen05 / cluster units dominate)
    with ThreadPoolExecutor(max_workers=max(1, min(len(sources()), os.cpu_count() or 1))) as ex:
        for src, obj, p in ex.map(compile_one, sources()):
            logs.append(f"== {os.path.basename(src)}\n{p.stderr}")
            if p.returncode != 0:
                sys.stderr.write(p.stdout + p.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            objs.append(obj)
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    tmp = LIB + ".tmp"
    link = [nvcc, *ARCH, "-shared", "-o", tmp, *objs, "-L", nccl_lib, "-l:libnccl.so.2", "-lcublas",
            "-Xlinker", f"-rpath={nccl_lib}"]
    if verbose:
        print(" ".join(link), flush=True)
    p = subprocess.run(link, capture_output=True, text=True)
    if p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    v = sys.argv[sys.argv.index("--variant") + 1] if "--variant" in sys.argv else ""
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, variant=v))
