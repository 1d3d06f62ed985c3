"""Run outputs (paper_2408_07609_b200.report) are byte-identical to the
reference's report writers (tests/golden/report/, made by
tests/golden/make_golden_report.py from blockswe.report): rasters of the
running maxima from the oracle (CPU) and from the device (GPU), the timing
CSV and the rank-cost CSV."""

import filecmp
import os

import numpy as np
import pytest

import systems
from conftest import GOLDEN

REPORT = os.path.join(GOLDEN, "report")
RUNS = (("quad_wetdry", 40), ("two_parent", 30))


def _compare_dir(got_dir, name):
    want_dir = os.path.join(REPORT, name)
    want = sorted(os.listdir(want_dir))
    got = sorted(os.listdir(got_dir))
    assert got == want
    for f in want:
        assert filecmp.cmp(os.path.join(got_dir, f), os.path.join(want_dir, f), shallow=False), f


@pytest.mark.parametrize("name,steps", RUNS)
def test_rasters_from_oracle_match_reference(oracle_mod, product, tmp_path, name, steps):
    from paper_2408_07609_b200 import report as R
    system, settings, _ = systems.make(product, name)
    sim = oracle_mod.OracleSimulation(system, settings)
    sim.run(steps)
    R.emit_rasters(system, sim.accumulators, str(tmp_path), tag="_golden")
    _compare_dir(str(tmp_path), name)


def test_raster_roundtrip(product, tmp_path):
    from paper_2408_07609_b200 import report as R
    path = os.path.join(REPORT, "quad_wetdry", "max_eta_L2_golden.txt")
    arr, head = R.read_raster(path)
    assert arr.shape == head[:2]
    out = tmp_path / "x.txt"
    with open(path) as f:
        header = f.readline().strip()
    R.write_raster(str(out), arr, header)
    assert filecmp.cmp(str(out), path, shallow=False)
    assert np.isnan(arr).any() or np.isfinite(arr).all()


def test_timing_and_rank_cost_csv(product, tmp_path):
    from paper_2408_07609_b200 import report as R
    rep = R.RunReport(steps=7, n_ranks=2, ranks=[
        R.RankTiming(0, {"mass": 0.125, "momentum": 1.0 / 3.0, "restrict": 2e-7}, 1.5),
        R.RankTiming(1, {"mass": 0.25, "halo-eta": 1e-3, "output": 0.0}, 2.25)])
    R.write_timing_csv(rep, str(tmp_path / "timing.csv"))
    assert filecmp.cmp(str(tmp_path / "timing.csv"), os.path.join(REPORT, "timing.csv"), shallow=False)
    cells = [50, 20, 70, 10, 40]
    plans = {"equal": product.equal_cell_plan(cells, 2), "split1": product.DecompositionPlan(tuple(cells), (1,))}
    R.write_rank_cost_csv(str(tmp_path / "rank_cost.csv"), plans, product.CostModel(slope=0.5, intercept=3.0))
    assert filecmp.cmp(str(tmp_path / "rank_cost.csv"), os.path.join(REPORT, "rank_cost.csv"), shallow=False)


@pytest.mark.gpu
@pytest.mark.parametrize("name,steps", RUNS)
def test_rasters_from_device_match_reference(cuda_device, product, tmp_path, name, steps):
    from paper_2408_07609_b200 import report as R
    system, settings, _ = systems.make(product, name)
    sim = product.Simulation(system, settings)
    sim.run(steps, threaded=False)
    R.emit_rasters(system, sim.accumulators, str(tmp_path), tag="_golden")
    _compare_dir(str(tmp_path), name)
