"""Build the in-tree CUDA library (sm_100a) with nvcc.

    python -m paper_2408_07609_b200.build

Flags: -fmad=false keeps the reference's (numpy's) unfused evaluation order
(SURVEY App. A); double division and sqrt are IEEE in CUDA; no fast math.
"""

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libtsunami_b200.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("step_kernels.cu", "api.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in ("common.cuh", "cbrt.cuh", "fastmath.cuh")] + [
    os.path.join(os.path.dirname(HERE), "include", "tsunami_b200.h")]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-fmad=false", "-Xptxas", "-v", "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
              "-shared", "-cudart", "static"]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    raise RuntimeError("nvcc not found")


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    cmd = [nvcc()] + NVCC_FLAGS + ["-o", LIB + ".tmp"] + SOURCES
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError("nvcc failed:\n" + res.stdout + res.stderr)
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(HERE, "ptxas.log"), "w") as f:
        f.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
