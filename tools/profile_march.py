"""Summarise an ncu capture of one step's march launches (Kochi-1.0, 1 GPU)
into profiles/: per launch its duration, DRAM traffic, issue and FP64-pipe
activity, and instruction counts per cell (all SASS, and the FP64-pipe
ones: DFMA/DMUL/DADD/DSETP/DMNMX) from the per-instruction source page.

    python tools/profile_march.py gpurun_out/X.ncu-rep profiles/r02/march_ncu.json

Runs here (no GPU): `ncu -i` reads the report.  Cells per launch follow the
library's width groups (csrc/api.cu create_impl)."""
import csv
import io
import json
import re
import subprocess
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

rep, out = sys.argv[1], sys.argv[2]
cmd = sys.argv[3] if len(sys.argv) > 3 else ("tools/ncu_kernel.sh (ncu --set full --clock-control none --import-source on "
                                             "-k regex:k_march --launch-skip 4 --launch-count 4 python "
                                             "tools/profile_step.py --steps 4)")


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True, check=True).stdout


def group_cells():
    """cells of each march template instance <W, TPC, MINB, PACKED>."""
    import paper_2408_07609_b200 as P
    s = P.build_kochi_scaled_config(1.0)
    cells = {}
    for _, b in s.all_blocks():
        L = b.nj + 3
        W = (L + 31) // 32 if L <= 128 else 4
        packed = 33 <= L <= 63 and ((128 // L) * L) / 128 > L / (32 * W) + 0.03
        key = (2, 1) if packed else (W, 0)
        cells[key] = cells.get(key, 0) + b.cell_count
    return cells


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr = raw[0]
col = {h: k for k, h in enumerate(hdr)}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size"]
units = raw[1]
kernels = []
for r in raw[2:]:
    name = r[col["Kernel Name"]]
    if "k_march" not in name:
        continue
    m = re.search(r"k_march<(\d+), (\d+), (\d+), (\d+)(?:, (\d+))?>", name)
    k = {"kernel": name.split("(")[0], "template": [int(x) for x in m.groups() if x is not None]}
    for w in want:
        v = r[col[w]].replace(",", "")
        k[w] = float(v) if v else None
        k.setdefault("units", {})[w] = units[col[w]]
    kernels.append(k)

# per-SASS thread instruction counts (source page)
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
fp64_ops = ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX")
cur, hdr2, sums = None, None, {}
for r in src:
    if r and r[0] == "Kernel Name":
        # the page lists every kernel twice; count its first listing
        cur = r[1] if r[1] not in sums else None
        if cur:
            sums[cur] = [0, 0]
        continue
    if r and r[0] == "Address":
        hdr2 = {h: k for k, h in enumerate(r)}
        continue
    if not cur or not hdr2 or len(r) < len(hdr2):
        continue
    try:
        n = int(r[hdr2["Thread Instructions Executed"]] or 0)
    except ValueError:
        continue
    op = re.sub(r"^@!?U?P[T0-9]\s+", "", r[hdr2["Source"]].strip()).split(" ")[0].split(".")[0]
    s = sums.setdefault(cur, [0, 0])
    s[0] += n
    if op in fp64_ops:
        s[1] += n

cells = group_cells()
tot_cells = tot_dp = tot_inst = tot_t = 0.0
for k in kernels:
    W, TPC, MINB, PK = k["template"][:4]
    c = cells.get((2, 1) if PK else (W, 0), 0)
    key = next((n for n in sums if re.sub(r"\(int\)|\(bool\)", "", n).startswith(k["kernel"].replace("void ", ""))
                or k["kernel"].replace("void ", "").replace(" ", "") in re.sub(r"\(int\)|\(bool\)", "", n).replace(" ", "")), None)
    ti, dp = sums.get(key, [0, 0])
    k.update({"cells": c, "thread_inst": ti, "dp_thread_inst": dp,
              "thread_inst_per_cell": ti / c if c else None, "dp_thread_inst_per_cell": dp / c if c else None})
    tot_cells += c
    tot_dp += dp
    tot_inst += ti
    tot_t += k["gpu__time_duration.sum"] or 0
res = {"report": os.path.basename(rep),
       "command": cmd,
       "cells": tot_cells, "thread_inst_per_cell": tot_inst / tot_cells, "dp_thread_inst_per_cell": tot_dp / tot_cells,
       "march_ms_serialised": tot_t, "kernels": kernels}
with open(out, "w") as f:
    json.dump(res, f, indent=1)
print(json.dumps({k: v for k, v in res.items() if k != "kernels"}, indent=1))
for k in kernels:
    print(k["template"], k["cells"], round(k["gpu__time_duration.sum"], 4), "ms", round(k["thread_inst_per_cell"] or 0, 1),
          "inst/cell", round(k["dp_thread_inst_per_cell"] or 0, 1), "dp/cell",
          k["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"], "% fp64")
