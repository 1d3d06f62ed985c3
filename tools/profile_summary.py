"""Write profiles/ summaries from a tools/gpu_profile.sh TAG run.

    python tools/profile_summary.py TAG [ROUND]     (reads gpurun_out/TAG_*; ROUND e.g. r02)
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
rnd = sys.argv[2] if len(sys.argv) > 2 else "r01"
title = {"r01": "Round 1", "r02": "Round 2"}.get(rnd, rnd)
G, PR = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")

rows = [r for r in csv.reader(open(os.path.join(G, f"{tag}_launches.csv"))) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    k = r[ki].split("(")[0]
    tot[k] += float(r[vi].replace(",", ""))
    cnt[k] += 1
S = sum(tot.values())
shutil.copy(os.path.join(G, f"{tag}_launches.csv"), os.path.join(PR, f"{rnd}_launches.csv"))
with open(os.path.join(PR, f"{rnd}_launches.md"), "w") as f:
    f.write(f"# {title} launch list (Kochi-1.0, 47,211,444 cells, 1 B200)\n\n")
    f.write("`ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --steps 3 "
            "--warmup 3 --no-cpu` (tools/gpu_profile.sh " + tag + "): 109 steps per kernel (3 warm-up, "
            "100 more inside the clock sampler's window, 3 timed, 3 end-to-end) plus the end-of-run "
            "accumulator fold of each run (`k_mass<1, 0>`) and the end-to-end leg's host-transfer repitch kernels.  Per step: one mass launch, "
            "four march launches (width groups W = 2, 1, 3 and the packed nj = 36 group) and the two merged "
            "exchange phases (`k_xops`: restriction + halo-eta, edges + prolongation + halo-flux). "
            "Cold-cache, serialised per-launch times; the raw list is `" + rnd + "_launches.csv`.\n\n")
    f.write("| kernel | launches | total µs | share | avg µs |\n|---|---|---|---|---|\n")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        f.write(f"| `{k}` | {cnt[k]} | {v / 1e3:.1f} | {v / S * 100:.1f} % | {v / cnt[k] / 1e3:.1f} |\n")

raw = subprocess.run(["ncu", "-i", os.path.join(G, f"{tag}_full.ncu-rep"), "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__block_size", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
keys = [k for k in keys if k in hdr]
stall = [k for k in hdr if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")]
kern = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    e = {"kernel": d["Kernel Name"].split("(")[0]}
    for k in keys:
        e[k] = float(d[k].replace(",", ""))
    e["units"] = {k: units[hdr.index(k)] for k in keys}
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(float(d[k].replace(",", "") or 0)) for k in stall}
    e["stall_samples_top"] = dict(sorted(st.items(), key=lambda x: -x[1])[:8])
    kern.append(e)
mom = [e for e in kern if "march" in e["kernel"]]
traffic = sum(e["dram__bytes_read.sum"] + e["dram__bytes_write.sum"] for e in mom) * 1e9
json.dump({"source": f"profiles/{rnd}_ncu_full.json (ncu --set full, Kochi-1.0, one step: the k_march launches)",
           "kernel": "k_march", "bytes_per_step": traffic}, open(os.path.join(PR, "momentum_traffic.json"), "w"),
          indent=1)
json.dump({"command": "tools/gpu_profile.sh: ncu --set full --clock-control none --import-source on "
                      "-k regex:'k_march|k_mass' --launch-skip 10 --launch-count 5 python bench.py --steps 2 "
                      "--warmup 3 --no-cpu", "kernels": kern},
          open(os.path.join(PR, f"{rnd}_ncu_full.json"), "w"), indent=1)
xrep = os.path.join(G, f"{tag}_xops.ncu-rep")
if os.path.exists(xrep):
    raw = subprocess.run(["ncu", "-i", xrep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    xr = list(csv.reader(raw.splitlines()))
    xo = []
    for r in xr[2:]:
        d = dict(zip(xr[0], r))
        xo.append({k: d[k] for k in ("Kernel Name", "Grid Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
                                     "dram__bytes_write.sum", "launch__registers_per_thread") if k in d}
                  | {"units": {k: xr[1][xr[0].index(k)] for k in ("gpu__time_duration.sum", "dram__bytes_read.sum",
                                                                   "dram__bytes_write.sum") if k in xr[0]}})
    json.dump({"command": "tools/gpu_profile.sh: ncu --set full -k regex:k_xops --launch-skip 4 --launch-count 2 "
                          "(one step's eta and flux phases)", "kernels": xo},
              open(os.path.join(PR, f"{rnd}_xops_ncu.json"), "w"), indent=1)
shutil.copy(os.path.join(G, f"{tag}_bench.json"), os.path.join(PR, f"{rnd}_bench_n1.json"))
shutil.copy(os.path.join(G, f"{tag}_ref.json"), os.path.join(PR, f"{rnd}_bench_ref.json"))
for e in kern:
    print(e["kernel"], e["gpu__time_duration.sum"], e["dram__bytes_read.sum"] + e["dram__bytes_write.sum"],
          e.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"))
print("momentum traffic/step", traffic)
