"""Build libsa.so in-tree with nvcc for sm_100a (no torch extension machinery)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libsa.so")
SO_TUNING = os.path.join(PKG, "libsa_tuning.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
]


# flat_scan_topk_kernel runs 352 threads at 1 CTA/SM: 65536 / 352 = 186 registers are
# available; let ptxas use them instead of spilling the epilogue's state.
PER_FILE_FLAGS = {"flat_scan.cu": ["-maxrregcount=184"]}


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp"))
                  + glob.glob(os.path.join(CSRC, "kernels", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
                  + glob.glob(os.path.join(CSRC, "*.h"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def needs_build(so: str = SO) -> bool:
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    return any(os.path.getmtime(f) > t for f in sources() + headers())


def build(force: bool = False, verbose: bool = False, tuning: bool = False) -> str:
    """Compile libsa.so.  tuning=True builds libsa_tuning.so instead: the same library with
    -DSA_TUNING_BUILD, which honours the timing-experiment switches (SA_EXPERIMENT, SA_NO_SEED,
    ...).  The product library never reads them; bench.py refuses the tuning
    library."""
    so = SO_TUNING if tuning else SO
    if not force and not needs_build(so):
        return so
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    objdir = os.path.join(PKG, "build_tuning" if tuning else "build")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    logs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.relpath(src, CSRC).replace(os.sep, "_") + ".o")
        extra = PER_FILE_FLAGS.get(os.path.basename(src), [])
        defs = ["-DSA_TUNING_BUILD"] if tuning else []
        cmd = [nvcc, *NVCC_FLAGS, *extra, *defs, "-I", os.path.join(ROOT, "include"), "-c", src,
               "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        logs.append(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        objs.append(obj)
    cmd = [nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", so, *objs,
           "-lcudart", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    with open(os.path.join(objdir, "ptxas.log"), "w") as f:
        f.write("\n".join(logs))
    if verbose:
        print("\n".join(logs))
    return so


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True, tuning="--tuning" in sys.argv)
