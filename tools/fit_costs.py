"""B200 per-cell step costs by block width (the balancer's cost table).

The reference fits a per-block GPU cost model from timed momentum calls
(balance.py:301-328, fit_cost_model).  Here the march's cost depends on the
block width (lanes per tile), so each width class is timed on its own:
a single-level system of identical, non-touching blocks of that width
(40 M cells: many waves, so the tail of the last wave is negligible), mass and momentum kernel times from
the library's per-step events.

    python tools/fit_costs.py [--widths 24,36,48,60,90]   (prints JSON)
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2408_07609_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--widths", default="24,36,48,60,90")
ap.add_argument("--cells", type=float, default=4e7)
ap.add_argument("--steps", type=int, default=40)
a = ap.parse_args()
out = {}
for nj in (int(w) for w in a.widths.split(",")):
    ni = 2400
    k = max(1, int(round(a.cells / (ni * nj))))
    dx = 30.0
    blocks = []
    for b in range(k):
        x0 = b * (ni + 12) * dx
        xs = x0 + (np.arange(ni) + 0.5) * dx
        h = np.broadcast_to((200.0 + 20.0 * np.sin(xs / 5000.0))[:, None], (ni, nj)).copy()
        blocks.append(P.Block(b + 1, (x0, 0.0), ni, nj, h))
    system = P.NestedGridSystem(levels=[P.GridLevel(1, dx, blocks)])
    span = k * (ni + 12) * dx
    settings = P.SimulationConfig(dt=0.2, initial=P.InitialCondition(
        "gaussian", 1.0, span / 6.0, (span / 2.0, nj * dx / 2.0)))
    sim = P.Simulation(system, settings)
    sim.run(5, threaded=False)
    sim.set_timing(True)
    sim.run(a.steps, threaded=False)
    m, mo, st = sim.kernel_seconds()
    cells = system.cell_count
    out[nj] = {"blocks": k, "cells": cells, "mass_ps_per_cell": m / cells * 1e12,
               "momentum_ps_per_cell": mo / cells * 1e12, "step_ps_per_cell": st / cells * 1e12}
    sim.close()
print(json.dumps(out))
