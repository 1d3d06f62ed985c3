"""Fit the B200 cost models the balancer uses, on the device:

* the reference-format per-block model (balance.measure_block_costs ->
  fit_cost_model -> save_cost_model; the B200 replacement of the
  reference's measure_momentum_cost, balance.py:301-328), and
* the per-width per-cell step table (balance.measure_width_costs) that
  packed_plan / phase_balanced_plan weigh blocks with.

    python tools/fit_costs.py OUTDIR [--widths 24,36,48,60,90] [--counts ...]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2408_07609_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("out")
ap.add_argument("--widths", default="24,36,48,60,90")
ap.add_argument("--counts", default="6000,24000,60000,240000,600000,1500000")
ap.add_argument("--repeats", type=int, default=3)
a = ap.parse_args()
os.makedirs(a.out, exist_ok=True)
samples = P.measure_block_costs([int(c) for c in a.counts.split(",")], repeats=a.repeats)
model = P.fit_cost_model(samples)
P.save_cost_model(model, os.path.join(a.out, "b200_cost_model.txt"))
table = P.measure_width_costs(tuple(int(w) for w in a.widths.split(",")))
P.save_width_costs(table, os.path.join(a.out, "b200_width_costs.json"))
print(json.dumps({"samples": samples, "model": model.__dict__, "widths": table}))
