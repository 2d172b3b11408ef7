"""Build libgfnx.so in-tree with nvcc for sm_100a (explicit -gencode, no torch arch list)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libgfnx.so")
BUILD = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
          "-I" + os.path.join(HERE, "..", "include")]
# (source, extra flags). check.cu must not contract FMAs (fp64 check mode = reference op order).
UNITS = [
    ("api.cu", []),
    ("check.cu", ["--fmad=false"]),
    ("fast.cu", ["-Xptxas", "-v"] if os.environ.get("GFNX_PTXAS_V") else []),
    ("lockstep.cu", ["-Xptxas", "-v"] if os.environ.get("GFNX_PTXAS_V") else []),
    ("group.cu", []),
    ("reward.cu", []),
    ("walk.cu", []),
    ("eb.cu", ["--fmad=false"]),
]
HOST_UNITS = ["host.cpp"]


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("command failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r.stdout + r.stderr


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(HERE, "..", "include", "gfnx.h"))
    objs, logs = [], []
    for src, extra in UNITS:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if _stale(o, [s] + headers):
            logs.append(_run([NVCC] + ARCH + COMMON + extra + ["-c", s, "-o", o]))
        objs.append(o)
    for src in HOST_UNITS:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if _stale(o, [s] + headers):
            logs.append(_run(["g++", "-std=c++17", "-O2", "-fPIC", "-ffp-contract=off", "-Wall",
                              "-I/usr/local/cuda/include", "-I" + os.path.join(HERE, "..", "include"),
                              "-c", s, "-o", o]))
        objs.append(o)
    if _stale(OUT, objs):
        logs.append(_run([NVCC] + ARCH + ["-shared", "-o", OUT] + objs + ["-ldl"]))
    if verbose:
        print("".join(logs))
    return OUT


if __name__ == "__main__":
    build(verbose="-v" in sys.argv)
    print(OUT)
