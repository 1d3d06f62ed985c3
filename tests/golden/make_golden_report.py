"""Golden output files from the REFERENCE's own report writers.

Runs the cbrt-aligned reference (see make_golden.py) on two fixture systems
and writes its rasters (blockswe.report.emit_rasters) and a timing / rank-cost
CSV of a fixed synthetic report into tests/golden/report/.  Runs only where
/root/reference exists; the files are committed.

    python tests/golden/make_golden_report.py
"""

import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, HERE)

import blockswe.grid as T                                   # noqa: E402
import blockswe.kernels as K                                # noqa: E402
from blockswe import report as R                            # noqa: E402
from blockswe.balance import CostModel, equal_cell_plan     # noqa: E402
from blockswe.runner import Simulation                      # noqa: E402

import oracle                                               # noqa: E402
import systems                                              # noqa: E402

OUT = os.path.join(HERE, "report")
RUNS = (("quad_wetdry", 40), ("two_parent", 30))


def main():
    K.np = oracle.CbrtAlignedNumpy()
    shutil.rmtree(OUT, ignore_errors=True)
    os.makedirs(OUT)
    for name, steps in RUNS:
        system, settings, _ = systems.make(T, name)
        plan = equal_cell_plan([b.cell_count for _, b in system.all_blocks()], 1)
        sim = Simulation(system, settings, plan)
        sim.run(steps, threaded=False)
        R.emit_rasters(system, sim.accumulators, os.path.join(OUT, name), tag="_golden")
    rep = R.RunReport(steps=7, n_ranks=2, ranks=[
        R.RankTiming(0, {"mass": 0.125, "momentum": 1.0 / 3.0, "restrict": 2e-7}, 1.5),
        R.RankTiming(1, {"mass": 0.25, "halo-eta": 1e-3, "output": 0.0}, 2.25)])
    R.write_timing_csv(rep, os.path.join(OUT, "timing.csv"))
    cells = [50, 20, 70, 10, 40]
    plans = {"equal": equal_cell_plan(cells, 2), "split1": equal_cell_plan(cells, 2).__class__(tuple(cells), (1,))}
    R.write_rank_cost_csv(os.path.join(OUT, "rank_cost.csv"), plans, CostModel(slope=0.5, intercept=3.0))
    print("wrote", OUT)


if __name__ == "__main__":
    main()
