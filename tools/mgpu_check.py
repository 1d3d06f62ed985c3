"""Multi-GPU parity check (run under torchrun, one process per GPU).

    torchrun --standalone --nproc-per-node 2 tools/mgpu_check.py [--system kochi] [--steps 40]

Runs the system decomposed over all ranks (blocks -> GPUs by an exact
min-max plan, exchanges over NVLink peer stores), gathers every block's
state on rank 0, runs the same system on rank 0's GPU alone and asserts
bitwise equality of eta/M/N and the running maxima.  Prints one JSON line.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2408_07609_b200 as P  # noqa: E402
from paper_2408_07609_b200 import distributed as D  # noqa: E402
import systems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--system", default="kochi")
ap.add_argument("--scale", type=float, default=0.001)
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--plan", default="minmax", choices=("minmax", "packed"))
args = ap.parse_args()

local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
if args.system == "kochi":
    system, settings, _ = systems.kochi(P, args.scale)
else:
    system, settings, _ = systems.make(P, args.system)
cells = [b.cell_count for _, b in system.all_blocks()]
plan = P.minmax_plan(cells, world) if args.plan == "minmax" else P.packed_plan(system, world)
sim = P.Simulation(system, settings, plan, distributed=True)
for chunk in (1, args.steps // 2, args.steps - 1 - args.steps // 2):
    sim.run(chunk, threaded=False)
mine = {bid: {f: getattr(st, f).copy() for f in ("eta_old", "eta_new", "m_old", "m_new", "n_old", "n_new")}
        for bid, st in sim.states.items()}
for bid, acc in sim.accumulators.items():
    mine[bid].update({f: getattr(acc, f).copy() for f in ("max_eta", "max_speed", "max_inundation")})
allf = D.gather_fields(mine, 0)
ok = True
bad = []
if rank == 0:
    ref = P.Simulation(system, settings, P.equal_cell_plan(cells, 1), distributed=False, device=local)
    for chunk in (1, args.steps // 2, args.steps - 1 - args.steps // 2):
        ref.run(chunk, threaded=False)
    for bid, fields in allf.items():
        st, acc = ref.states[bid], ref.accumulators[bid]
        for f, v in fields.items():
            r = getattr(acc, f) if f.startswith("max") else getattr(st, f)
            if not np.array_equal(v, r, equal_nan=True):
                ok = False
                bad.append((bid, f, float(np.nanmax(np.abs(v - r)))))
    print(json.dumps({"system": args.system, "ranks": world, "steps": args.steps, "plan": args.plan, "owners": [plan.rank_of(k) for k in range(plan.n_blocks)],
                      "blocks": len(cells), "bitwise_equal_to_1gpu": ok, "diffs": bad[:5]}), flush=True)
ok = D.first_error(None if ok else ("mismatch",))
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok is None else 1)
