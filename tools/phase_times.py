"""Per-phase device time of one step on every rank (first graph step's
phase events), Kochi-1.0.

    torchrun --nproc-per-node N tools/phase_times.py
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2408_07609_b200 as P  # noqa: E402
from paper_2408_07609_b200 import _native as N  # noqa: E402
from paper_2408_07609_b200 import distributed as D  # noqa: E402

local = int(os.environ.get("LOCAL_RANK", "0"))
world = int(os.environ.get("WORLD_SIZE", "1"))
torch.cuda.set_device(local)
if world > 1:
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
scale = float(os.environ.get("KOCHI_SCALE", "1.0"))
system = P.build_kochi_scaled_config(scale)
settings = P.kochi_settings(system)
cells = [b.cell_count for _, b in system.all_blocks()]
plan = P.packed_plan(system, world) if world > 1 else None
sim = P.Simulation(system, settings, plan, device=local)
sim.run(5, threaded=False)
out = []
for _ in range(2):
    sim.run(20, threaded=False)
    buf = (ctypes.c_double * 7)()
    tot = ctypes.c_double()
    N.check(N.lib().ts_timings(sim._h, buf, ctypes.byref(tot)))
    # per step: routines of the run are apportioned from its first graph
    # step's phase events over the run's device total
    out.append({k: round(v * 1e6 / 20, 1) for k, v in zip(P.ROUTINES, buf)} | {"step_us": round(tot.value * 1e6 / 20, 1)})
res = {"rank": sim.rank, "steps": out}
if world > 1:
    import pickle
    allr = [pickle.loads(b) for b in D.all_gather_bytes(pickle.dumps(res))]
else:
    allr = [res]
if sim.rank == 0:
    for r in allr:
        print(json.dumps(r))
sim.close()
if world > 1:
    dist.barrier()
    dist.destroy_process_group()
