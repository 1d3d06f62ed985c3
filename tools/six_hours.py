"""The BASELINE.json headline run: a 6-hour simulation (108,000 steps of
0.2 s) of the 47.2 M-cell 5-level Kochi domain on one GPU, timed end to
end (setup excluded, device time by events around the run).  Prints one
JSON line with the wall / device time and a summary of the maxima.

    python tools/six_hours.py [--steps 108000] [--scale 1.0]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2408_07609_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=108_000)
ap.add_argument("--scale", type=float, default=1.0)
a = ap.parse_args()
world = int(os.environ.get("WORLD_SIZE", "1"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
if world > 1:                      # torchrun: one process per GPU, packed plan
    import torch.distributed as dist
    from paper_2408_07609_b200 import distributed as D
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
system = P.build_kochi_scaled_config(a.scale)
settings = P.kochi_settings(system)
sim = P.Simulation(system, settings, device=local)
ext = torch.cuda.ExternalStream(sim.stream_ptr)
if world > 1:
    dist.barrier()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
e0.record(ext)
status = "ok"
try:
    rep = sim.run(a.steps, threaded=False)
except P.NumericsError as exc:
    status = f"NumericsError: {exc}"
e1.record(ext)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
dev = e0.elapsed_time(e1) / 1e3
summary = {}
for lvl in system.levels:
    mine = [b for b in lvl.blocks if b.block_id in sim.accumulators]
    me = [float(np.nanmax(sim.accumulators[b.block_id].max_eta)) for b in mine] or [float("-inf")]
    ms = [float(np.nanmax(sim.accumulators[b.block_id].max_speed)) for b in mine] or [float("-inf")]
    summary[f"L{lvl.level_index}"] = {"max_eta": max(me), "max_speed": max(ms)}
if world > 1:
    wall, dev = D.max_over_ranks(wall), D.max_over_ranks(dev)
    import pickle
    parts = [pickle.loads(x) for x in D.all_gather_bytes(pickle.dumps(summary))]
    summary = {k: {f: max(p[k][f] for p in parts) for f in ("max_eta", "max_speed")} for k in summary}
if sim.rank == 0:
    print(json.dumps({"steps": a.steps, "simulated_s": a.steps * settings.dt, "cells": system.cell_count,
                      "gpus": world, "status": status, "wall_s": wall, "device_s": dev,
                      "gcell_per_s": system.cell_count * a.steps / dev / 1e9, "levels": summary}))
sim.close()
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
