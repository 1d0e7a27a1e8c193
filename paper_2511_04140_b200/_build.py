"""Build libfalcon_b200.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

Objects are compiled in parallel and cached under build/ by source mtime; the shared
library links the CUDA runtime statically so it loads beside torch's own runtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "falcon_b200")
LIB = os.path.join(PKG, "libfalcon_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

# -fmad=false: no multiply/add contraction anywhere -- every FP result must match the
# CPU reference bit for bit (the kernels also use explicit __dmul_rn/__ddiv_rn).
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-fmad=false",
         "-std=c++17", "-Xcompiler", "-fPIC,-O2", "-I", os.path.join(ROOT, "include")]
UNITS = ["kernels_all.cu", "capi.cu", "runtime.cu", "pipeline.cu", "gds.cu"]
HEADERS = ["falcon_common.cuh", "kernels.h", "runtime.h", "encode.cu", "decode.cu", "tables.cu", "selftest.cu",
           "synth.cu", "field.cuh", "dpds.cuh", "launch_cache.cuh"]


def _mtime(p: str) -> float:
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(verbose: bool = False, force: bool = False, defines: tuple = (), out: str | None = None) -> str:
    """Build the library; `defines` + `out` make a variant (own object dir, own .so) for
    A/B kernel experiments."""
    build_dir = BUILD if not defines else os.path.join(ROOT, "build", "variant_" + "_".join(d.replace("=", "") for d in defines))
    lib = out or LIB
    flags = FLAGS + [f"-D{d}" for d in defines]
    os.makedirs(build_dir, exist_ok=True)
    dep = max([_mtime(os.path.join(CSRC, h)) for h in HEADERS] +
              [_mtime(os.path.join(ROOT, "include", "falcon_b200.h")), _mtime(__file__)])
    objs, jobs = [], []
    for u in UNITS:
        src = os.path.join(CSRC, u)
        obj = os.path.join(build_dir, u.replace(".cu", ".o"))
        objs.append(obj)
        if force or _mtime(obj) < max(_mtime(src), dep):
            jobs.append([NVCC, *flags, "-c", src, "-o", obj] + (["-Xptxas", "-v"] if verbose else []))

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("nvcc failed:\n" + " ".join(cmd) + "\n" + r.stdout + r.stderr)
        return r.stdout + r.stderr

    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for out in ex.map(run, jobs):
            if verbose and out:
                print(out)
    if force or jobs or _mtime(lib) < max(_mtime(o) for o in objs):
        run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
             "-o", lib, *objs, "-lpthread", "-ldl"])
    return lib


if __name__ == "__main__":
    import sys
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
