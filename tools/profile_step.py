"""Run a few steps of a workload for ncu (kernels are profiled per graph node).

    python tools/profile_step.py [--config kochi] [--scale 1.0] [--steps 3]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2408_07609_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="kochi")
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--steps", type=int, default=3)
a = ap.parse_args()
system, settings, label = bench.build_workload(P, a.config, a.scale)
sim = P.Simulation(system, settings)
sim.run(a.steps, threaded=False)
print(label, "ok", sim.launches_per_step, "launches/step")
