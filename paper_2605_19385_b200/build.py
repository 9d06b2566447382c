"""Build the in-tree shared library paper_2605_19385_b200/liblbx.so (sm_100a only).

nvcc -gencode arch=compute_100a,code=sm_100a (plain -arch=sm_100a silently targets sm_100 in this
toolchain and tcgen05 fails to assemble).  CUDA runtime linked statically, the
driver API (cuTensorMapEncodeTiled) resolved at run time through cudaGetDriverEntryPoint, so the
.so has no dependency beyond libc/libstdc++ and the driver.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "liblbx.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(f for f in os.listdir(CSRC) if f.endswith((".cu", ".cpp")))


def _flags():
    return ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-Wall,-fvisibility=hidden",
                   "--expt-relaxed-constexpr",
                   "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-Xptxas", "-v" if os.environ.get("LBX_PTXAS_V") else "-O3"] + \
        os.environ.get("LBX_EXTRA_NVCC_FLAGS", "").split()  # experiments only (A/B builds)


def _compile(src: str) -> str:
    out = os.path.join(OBJ, src + ".o")
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    deps += [os.path.join(ROOT, "include", "lbx", f) for f in os.listdir(os.path.join(ROOT, "include", "lbx"))]
    srcp = os.path.join(CSRC, src)
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(p) for p in deps + [srcp]):
        return out
    cmd = [nvcc()] + _flags() + ["-c", srcp, "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if os.environ.get("LBX_PTXAS_V"):
        sys.stderr.write(r.stderr)
    return out


def build(verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, sources()))
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + ["-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
        os.replace(LIB + ".tmp", LIB)
    if verbose:
        print(LIB)
    return LIB




def build_tools(verbose: bool = False) -> str:
    """tools/c5_replay (config-5 trace replay harness), linked against the in-tree liblbx.so."""
    tools = os.path.join(ROOT, "tools")
    out = os.path.join(tools, "c5_replay")
    srcs = [os.path.join(tools, f) for f in ("c5_replay.cpp", "lb_sim.cpp")]
    deps = srcs + [os.path.join(tools, "lb_sim.hpp"), LIB]
    if os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(p) for p in deps):
        return out
    cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"), "-I", tools] + srcs + [
        "-L", HERE, "-llbx", "-Wl,-rpath,$ORIGIN/../paper_2605_19385_b200", "-lpthread", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"c5_replay build failed:\n{r.stderr}")
    if verbose:
        print(out)
    return out


if __name__ == "__main__":
    build(verbose=True)
    build_tools(verbose=True)
