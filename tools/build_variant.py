"""Build an experimental copy of the library with extra nvcc -D flags.

    python tools/build_variant.py NAME [-DFOO=1 ...]   ->  variants/lib_NAME.so

Select it at run time with TSUNAMI_B200_LIB=variants/lib_NAME.so.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2408_07609_b200 import build as B  # noqa: E402

name, extra = sys.argv[1], sys.argv[2:]
os.makedirs(os.path.join(ROOT, "variants"), exist_ok=True)
out = os.path.join(ROOT, "variants", f"lib_{name}.so")
flags = [f for f in B.NVCC_FLAGS if f != "-v"]
flags = [f for i, f in enumerate(flags) if not (f == "-Xptxas" and i + 1 < len(flags) and flags[i + 1] == "-v")]
res = subprocess.run([B.nvcc()] + B.NVCC_FLAGS + extra + ["-o", out] + B.SOURCES, capture_output=True, text=True)
if res.returncode:
    sys.exit(res.stdout + res.stderr)
with open(out + ".ptxas.log", "w") as f:
    f.write(res.stderr)
print(out)
