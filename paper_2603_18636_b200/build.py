"""Build libcoclust.so (sm_100a) in-tree with nvcc.

    python -m paper_2603_18636_b200.build [--force] [--verbose]

Every translation unit is compiled with `-gencode arch=compute_100a,code=sm_100a -lineinfo -O3`;
the CUDA runtime is linked statically so the library only needs the driver at run time.
"""
from __future__ import annotations

import argparse
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
# variant builds for A/B experiments: CS_VARIANT=name CS_EXTRA_FLAGS="-DFOO" -> libcoclust_name.so
VARIANT = os.environ.get("CS_VARIANT", "")
LIB = os.path.join(HERE, f"libcoclust_{VARIANT}.so" if VARIANT else "libcoclust.so")
BUILD = os.path.join(HERE, f"_build_{VARIANT}" if VARIANT else "_build")
SOURCES = ["api.cu", "cluster.cu", "assign.cu", "select.cu", "attn.cu", "profile.cu", "peer.cu"]
HEADERS = ["common.cuh", "kernels.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include")] + os.environ.get("CS_EXTRA_FLAGS", "").split()


def _digest(paths):
    h = hashlib.sha256()
    for p in paths:
        with open(p, "rb") as f:
            h.update(f.read())
    h.update(" ".join(FLAGS).encode())
    return h.hexdigest()


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "coclust.h")]
    objs = []
    for src in SOURCES:
        sp = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src.replace(".cu", ".o"))
        stamp = obj + ".sha"
        dig = _digest([sp] + hdrs)
        if force or not os.path.exists(obj) or not os.path.exists(stamp) or open(stamp).read() != dig:
            cmd = [NVCC, *FLAGS, "-c", sp, "-o", obj]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                sys.stderr.write(r.stdout + r.stderr)
                raise RuntimeError(f"nvcc failed on {src}")
            if verbose:
                sys.stderr.write(r.stderr)
            with open(stamp, "w") as f:
                f.write(dig)
        objs.append(obj)
    newest = max(os.path.getmtime(o) for o in objs)
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
               "-o", LIB, *objs]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError("nvcc link failed")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
