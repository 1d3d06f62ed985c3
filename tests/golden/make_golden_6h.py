"""6-hour golden: the cbrt-aligned REFERENCE on Kochi-0.001 (47,211 cells,
5 levels, 84 blocks) for 108,000 steps (dt 0.2 s), dumped as digests plus
accumulator arrays (at the last good checkpoint when the reference fails).  Runs only where /root/reference exists; takes ~2 h.

    python tests/golden/make_golden_6h.py
"""
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, HERE)

import blockswe.grid as T                      # noqa: E402
import blockswe.kernels as K                   # noqa: E402
from blockswe.balance import equal_cell_plan   # noqa: E402
from blockswe.runner import Simulation         # noqa: E402

import oracle                                  # noqa: E402
import systems                                 # noqa: E402

STEPS = 108_000

K.np = oracle.CbrtAlignedNumpy()
system, settings, _ = systems.kochi(T, 0.001)
plan = equal_cell_plan([b.cell_count for _, b in system.all_blocks()], 1)
sim = Simulation(system, settings, plan)
t0 = time.time()
checkpoints = {}
failure = None
done = 0


def checkpoint(target):
    checkpoints[str(target)] = {f"{bid}/{f}": systems.digest(getattr(st, f))
                                for bid, st in sim.states.items() for f in ("eta_old", "m_old", "n_old")}
    checkpoints[str(target)].update({f"{bid}/{f}": systems.digest(getattr(sim.accumulators[bid], f))
                                     for bid in sim.states for f in ("max_eta", "max_speed", "max_inundation")})


# digests at 1000/10000/36000 steps, then 1000-step chunks: the reference
# itself blows up on this system a little after step 37,000, so the golden
# records the last good checkpoint and the failing chunk + message
targets = [1000, 10000, 36000] + list(range(37000, STEPS + 1, 1000))
for target in targets:
    try:
        sim.run(target - done, threaded=False)
    except K.NumericsError as e:
        failure = {"after": done, "within": target - done, "message": str(e)}
        print("failure", failure, flush=True)
        break
    done = target
    checkpoint(target)
    last_acc = {f"{bid}/{f}": getattr(sim.accumulators[bid], f).copy()
                for bid in sim.states for f in ("max_eta", "max_inundation")}
    print(target, "steps", round(time.time() - t0), "s", flush=True)
out = {"steps": STEPS, "ranks": 1, "failure": failure, "last_good": done,
       "eta0": {str(b): systems.digest(e) for b, e in systems.eta0_of(system, settings).items()},
       "h": {str(b.block_id): systems.digest(b.h) for _, b in system.all_blocks()},
       "checkpoints": checkpoints, "wall_s": time.time() - t0}
with open(os.path.join(HERE, "kochi6h.json"), "w") as f:
    json.dump(out, f, indent=0)
np.savez_compressed(os.path.join(HERE, "kochi6h_acc.npz"), **last_acc)   # at the last good step
