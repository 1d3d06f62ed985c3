"""Per-launch device time of one Kochi-1.0 step on every rank
(ts_trace_step: one captured step with an event after every launch, the
width groups' march launches serialised), averaged over a few steps.

    python tools/trace_step.py [--steps 4] [--scale 1.0]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/trace_step.py
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2408_07609_b200 as P  # noqa: E402
from paper_2408_07609_b200 import _native as N  # noqa: E402
from paper_2408_07609_b200 import distributed as D  # noqa: E402

KINDS = {0: "mass", 1: "restrict-src", 2: "restrict-2nd", 3: "halo-eta", 4: "barrier", 5: "restrict-recv",
         6: "halo-eta-2", 7: "march", 8: "edges", 9: "prolong-src", 10: "prolong-2nd", 11: "prolong-recv",
         12: "halo-flux", 13: "eta-phase", 14: "flux-phase"}

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--warmup", type=int, default=6)
ap.add_argument("--scale", type=float, default=1.0)
a = ap.parse_args()
local = int(os.environ.get("LOCAL_RANK", "0"))
world = int(os.environ.get("WORLD_SIZE", "1"))
torch.cuda.set_device(local)
dist = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
system = P.build_kochi_scaled_config(a.scale)
settings = P.kochi_settings(system)
counts = [b.cell_count for _, b in system.all_blocks()]
plan = P.packed_plan(system, world) if world > 1 else P.equal_cell_plan(counts, 1)
sim = P.Simulation(system, settings, plan, device=local, distributed=world > 1)
sim.run(a.warmup, threaded=False)
lib = N.lib()
cap = 96
acc = {}
order = []
for _ in range(a.steps):
    lab = (ctypes.c_int32 * cap)()
    us = (ctypes.c_float * cap)()
    cnt = ctypes.c_int32()
    N.check(lib.ts_trace_step(sim._h, lab, us, cap, ctypes.byref(cnt)))
    seen = {}
    for k in range(min(cnt.value, cap)):
        kind, grp = divmod(lab[k], 16)
        name = KINDS.get(kind, str(kind)) + (f"[{grp}]" if kind in (7, 4) else "")
        seen[name] = seen.get(name, 0) + 1
        key = f"{name}#{seen[name]}"
        if key not in acc:
            acc[key] = 0.0
            order.append(key)
        acc[key] += us[k]
res = {"rank": sim.rank, "launches": [(k, round(acc[k] / a.steps, 1)) for k in order],
       "step_us": round(sum(acc.values()) / a.steps, 1)}
if world > 1:
    import pickle
    allr = [pickle.loads(b) for b in D.all_gather_bytes(pickle.dumps(res))]
else:
    allr = [res]
if sim.rank == 0:
    print(json.dumps({"world": world, "scale": a.scale, "ranks": allr}))
sim.close()
if dist is not None:
    dist.barrier()
    dist.destroy_process_group()
