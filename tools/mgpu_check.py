"""Multi-GPU parity check (run under torchrun, one process per GPU).

    torchrun --standalone --nproc-per-node 2 tools/mgpu_check.py [--system kochi] [--steps 40]

More processes than GPUs share the GPUs round-robin (an 8-rank check runs on
a 4-GPU box).

Runs the system decomposed over all ranks (blocks -> GPUs by an exact
min-max or the packed plan, exchanges over NVLink peer stores), gathers
every block's state on rank 0, runs the same system and plan on rank 0's
GPU alone (one process, the plan's apply order) and asserts bitwise
equality of eta/M/N and the running maxima.  Prints one JSON line per
system (``--system fuzz``: per random nested system).
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
ap.add_argument("--system", default="kochi",
                help="a systems.py name, kochi, fuzz (random_nested seeds), or nan (a failing run)")
ap.add_argument("--scale", type=float, default=0.001)
ap.add_argument("--steps", type=int, default=40)
ap.add_argument("--plan", default="minmax", choices=("minmax", "packed"))
ap.add_argument("--seeds", type=int, default=12, help="--system fuzz: seeds 0..N-1 with >= ranks blocks")
args = ap.parse_args()

FIELDS = ("eta_old", "eta_new", "m_old", "m_new", "n_old", "n_new")
ACCS = ("max_eta", "max_speed", "max_inundation")

local = int(os.environ.get("LOCAL_RANK", "0"))
# more ranks than GPUs (e.g. an 8-rank check on a 4-GPU box): ranks share
# GPUs round-robin (CUDA IPC works within a device; the contexts time-slice)
local = local % max(1, torch.cuda.device_count())
torch.cuda.set_device(local)
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()


def check(system, settings, steps, name):
    """Decomposed run vs rank 0's 1-GPU run; rank 0 prints a JSON line."""
    cells = [b.cell_count for _, b in system.all_blocks()]
    plan = P.minmax_plan(cells, world) if args.plan == "minmax" else P.packed_plan(system, world)
    chunks = (1, steps // 2, steps - 1 - steps // 2)
    sim = P.Simulation(system, settings, plan, distributed=True, device=local)
    for chunk in chunks:
        sim.run(chunk, threaded=False)
    mine = {bid: {f: getattr(st, f).copy() for f in FIELDS} for bid, st in sim.states.items()}
    for bid, acc in sim.accumulators.items():
        mine[bid].update({f: getattr(acc, f).copy() for f in ACCS})
    sim.close()
    allf = D.gather_fields(mine, 0)
    ok, bad = True, []
    if rank == 0:
        # the same plan in one process: the reference's apply order (which
        # rank's halo / coupling write lands last where writes overlap)
        ref = P.Simulation(system, settings, plan, distributed=False, device=local)
        for chunk in chunks:
            ref.run(chunk, threaded=False)
        for bid, fields in allf.items():
            st, acc = ref.states[bid], ref.accumulators[bid]
            for f, v in fields.items():
                r = getattr(acc, f) if f.startswith("max") else getattr(st, f)
                if not np.array_equal(v, r, equal_nan=True):
                    ok = False
                    bad.append((bid, f, float(np.nanmax(np.abs(v - r)))))
        ref.close()
        print(json.dumps({"system": name, "ranks": world, "steps": steps, "plan": args.plan,
                          "owners": [plan.rank_of(k) for k in range(plan.n_blocks)],
                          "blocks": len(cells), "bitwise_equal_to_1gpu": ok, "diffs": bad[:5]}), flush=True)
    return ok


def check_failure(steps):
    """A NaN depth on the last rank's block: every rank stops with the same
    exception and message as the one-process run of the same plan."""
    blocks = [systems.flat_block(P, k + 1, (80.0 * k, 0.0), 8, 8, 30.0) for k in range(world - 1)]
    blocks.append(P.Block(world, (80.0 * (world - 1), 0.0), 8, 8, np.where(np.eye(8, dtype=bool), np.nan, 30.0)))
    system = P.NestedGridSystem(levels=[P.GridLevel(1, 10.0, blocks)])
    settings = P.SimulationConfig(dt=0.2)
    plan = P.equal_cell_plan([b.cell_count for _, b in system.all_blocks()], world)

    def outcome(sim):
        try:
            sim.run(steps, threaded=False)
            return ("ok", "")
        except Exception as exc:          # noqa: BLE001 - the type is the result
            return (type(exc).__name__, str(exc))

    sim = P.Simulation(system, settings, plan, distributed=True, device=local)
    mine = outcome(sim)
    sim.close()
    outs = [None] * world
    dist.all_gather_object(outs, mine)
    ok = True
    if rank == 0:
        ref = P.Simulation(system, settings, plan, distributed=False, device=local)
        want = outcome(ref)
        ref.close()
        ok = want[0] == "NumericsError" and all(o == want for o in outs)
        print(json.dumps({"system": "nan_last_rank", "ranks": world, "steps": steps, "one_process": want,
                          "ranks_raised": outs, "bitwise_equal_to_1gpu": ok, "diffs": []}), flush=True)
    return ok


ok = True
if args.system == "nan":
    ok = check_failure(args.steps)
elif args.system == "kochi":
    system, settings, _ = systems.kochi(P, args.scale)
    ok = check(system, settings, args.steps, "kochi")
elif args.system == "fuzz":
    for seed in range(args.seeds):
        system, settings, n, _ = systems.random_nested(P, seed)
        if system.n_blocks >= world:
            ok = check(system, settings, args.steps, f"fuzz{seed}") and ok
else:
    system, settings, _ = systems.make(P, args.system)
    ok = check(system, settings, args.steps, args.system)
ok = D.first_error(None if ok else ("mismatch",))
dist.barrier()
dist.destroy_process_group()
sys.exit(0 if ok is None else 1)
