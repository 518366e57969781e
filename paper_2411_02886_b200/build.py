"""In-tree build of the native library: paper_2411_02886_b200/_build/libtokenselect.so.

Every .cu is compiled for sm_100a only (``-gencode arch=compute_100a,code=sm_100a``)
with ``-lineinfo`` so ncu source pages map back to the kernels; the host C-ABI
layer (abi.cpp) is compiled by nvcc too and the CUDA runtime is linked
statically, so the .so travels to the GPU box with no extra dependencies.

    python -m paper_2411_02886_b200.build        # incremental
    python -m paper_2411_02886_b200.build --force
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_build")
LIB = os.path.join(OUT, "libtokenselect.so")
ROOT = os.path.dirname(HERE)

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
          "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]

SOURCES = ["decode.cu", "step.cu", "vote.cu", "util.cu", "aux.cu", "prefill.cu", "prefill_tc.cu", "comm.cpp", "abi.cpp"]
HEADERS = ["common.cuh", "params.h", "decode.h", "aux.h", "step.h", "vote.h", "util.h", "comm.h"]


def _newer(src_paths, target):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(p) > t for p in src_paths)


def _compile(src, force):
    path = os.path.join(CSRC, src)
    obj = os.path.join(OUT, src + ".o")
    deps = [path] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "tokenselect.h")]
    if not force and not _newer(deps, obj):
        return obj, None
    lang = ["-x", "cu"] if src.endswith(".cu") else ["-x", "c++"]
    cmd = [NVCC] + ARCH + COMMON + lang + ["-c", path, "-o", obj] + os.environ.get("TS_NVCC_FLAGS", "").split()
    if src.endswith(".cu"):
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(lambda s: _compile(s, force), SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for (_, log), s in zip(results, SOURCES):
            if log:
                print(f"--- {s}\n{log}", file=sys.stderr)
    # relink only when an object (or nothing) changed
    if force or _newer(objs, LIB):
        cmd = [NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-lrt", "-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose))
