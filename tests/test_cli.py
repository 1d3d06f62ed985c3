"""The command line against the reference's own CLI expectations
(/root/reference/pkg/tests/test_cli.py: exit codes, outputs, plan files,
snapshots, traces, failure markers, level budgets; cli.py:28-290), plus the
per-phase message counts of the synthesised trace
(pkg/tests/test_exchange.py:230-260).  ``main`` runs in-process; the
``run`` cases need the GPU."""

import os

import numpy as np
import pytest

from paper_2408_07609_b200.__main__ import main

GOOD_CONFIG = """\
dt: 0.2
duration: 4.0
initial: {kind: gaussian, amplitude: 0.4, sigma: 60.0, center: [120.0, 60.0]}
levels:
  - dx: 10.0
    blocks:
      - {id: 1, origin: [0.0, 0.0], ni: 12, nj: 12, bathymetry: 40.0}
      - {id: 2, origin: [120.0, 0.0], ni: 12, nj: 12, bathymetry: 40.0}
"""

BAD_CONFIG = """\
dt: 0.2
levels:
  - dx: 10.0
    blocks:
      - {id: 1, origin: [0.0, 0.0], ni: 6, nj: 6, bathymetry: 500.0}
"""

BUDGET_CONFIG = """\
dt: 0.2
rank_budgets: [2, 1]
initial: {kind: gaussian, amplitude: 0.2, sigma: 40.0, center: [54.0, 27.0]}
levels:
  - dx: 9.0
    blocks:
      - {id: 1, origin: [0.0, 0.0], ni: 6, nj: 6, bathymetry: 8.0}
      - {id: 2, origin: [54.0, 0.0], ni: 6, nj: 6, bathymetry: 8.0}
  - dx: 3.0
    blocks:
      - {id: 3, origin: [18.0, 9.0], ni: 18, nj: 12, bathymetry: 8.0}
"""


@pytest.fixture
def good_config(tmp_path):
    p = tmp_path / "good.yaml"
    p.write_text(GOOD_CONFIG)
    return str(p)


@pytest.fixture
def bad_config(tmp_path):
    p = tmp_path / "bad.yaml"
    p.write_text(BAD_CONFIG)
    return str(p)


# ---------------------------------------------------------------- CPU only
def test_validate_ok_and_cfl_exit_code(good_config, bad_config, capsys):
    assert main(["validate", "--config", good_config]) == 0
    assert "all checks passed" in capsys.readouterr().out
    assert main(["validate", "--config", bad_config]) == 2
    assert "cfl" in capsys.readouterr().out


def test_run_refuses_invalid_config(bad_config, tmp_path):
    assert main(["run", "--config", bad_config, "--steps", "5", "--out", str(tmp_path / "x")]) == 2


def test_unknown_decomp_is_runtime_error(good_config, tmp_path):
    assert main(["run", "--config", good_config, "--steps", "1", "--decomp", "bogus",
                 "--out", str(tmp_path / "x")]) == 1


def test_plan_builders(good_config, tmp_path):
    """--decomp equal / opt / packed / file: and per-level budgets map onto
    the plans the reference builds (cli.py:107-133)."""
    import argparse
    from paper_2408_07609_b200 import __main__ as M
    from paper_2408_07609_b200.config import load_config
    system, settings = load_config(good_config)
    ns = argparse.Namespace(decomp="equal", model="ref", seed=0)
    eq = M._build_plan(ns, system, settings, 2)
    assert eq.separators == (1,)
    ns.decomp = "opt"
    assert M._build_plan(ns, system, settings, 2).separators == (1,)
    ns.decomp = "packed"
    assert sorted(M._build_plan(ns, system, settings, 2).owners) == [0, 1]
    f = tmp_path / "plan.txt"
    M._save_plan(str(f), eq)
    assert f.read_text().startswith("# separator positions")
    ns.decomp = f"file:{f}"
    assert M._build_plan(ns, system, settings, 2).separators == (1,)
    with pytest.raises(ValueError):
        M._build_plan(ns, system, settings, 3)
    p = tmp_path / "budget.yaml"
    p.write_text(BUDGET_CONFIG)
    system, settings = load_config(str(p))
    ns.decomp = "equal"
    assert M._build_plan(ns, system, settings, 3).separators == (1, 2)   # one rank per parent block


def test_balance_fit_from_samples_and_model_file(tmp_path, capsys):
    import paper_2408_07609_b200 as P
    xs = np.linspace(1e4, 2e6, 50)
    rows = np.stack([xs, 1.09e-4 * xs + 46.2], axis=1)
    csv_path = tmp_path / "samples.csv"
    np.savetxt(csv_path, rows, delimiter=",")
    out = tmp_path / "fit"
    assert main(["balance", "fit", "--samples", str(csv_path), "--out", str(out)]) == 0
    text = (out / "model.txt").read_text()
    assert "slope" in text and "intercept" in text
    assert "R^2 = 1.0000" in capsys.readouterr().out
    m = P.load_cost_model(str(out / "model.txt"))
    assert abs(m.slope - 1.09e-4) < 1e-12 and abs(m.intercept - 46.2) < 1e-6
    assert main(["balance", "fit", "--out", str(tmp_path)]) == 1           # needs a source


def test_model_file_matches_reference_format(tmp_path):
    """save_cost_model / load_cost_model read and write the reference's file
    (balance.py:77-94) in both directions."""
    import sys
    import paper_2408_07609_b200 as P
    from conftest import REFERENCE_SRC
    m = P.CostModel(slope=4.2e-5, intercept=1.25, r_squared=0.99)
    P.save_cost_model(m, str(tmp_path / "a.txt"))
    assert P.load_cost_model(str(tmp_path / "a.txt")) == m
    if os.path.isdir(REFERENCE_SRC):
        sys.path.insert(0, REFERENCE_SRC)
        from blockswe import balance as RB
        r = RB.load_cost_model(str(tmp_path / "a.txt"))
        assert (r.slope, r.intercept, r.r_squared) == (m.slope, m.intercept, m.r_squared)
        RB.save_cost_model(r, str(tmp_path / "b.txt"))
        assert P.load_cost_model(str(tmp_path / "b.txt")) == m


def test_balance_optimize(tmp_path, capsys):
    cfg = os.path.join(os.path.dirname(__file__), "golden", "configs", "cfg2.yaml")
    out = tmp_path / "opt"
    assert main(["balance", "optimize", "--config", cfg, "--ranks", "2", "--out", str(out)]) == 0
    assert (out / "separators.txt").exists() and (out / "rank_costs.csv").exists()
    assert "->" in capsys.readouterr().out
    assert main(["balance", "optimize", "--config", cfg, "--ranks", "1", "--level", "9",
                 "--out", str(out)]) == 1


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_run_writes_outputs(cuda_device, good_config, tmp_path):
    out = tmp_path / "out"
    assert main(["run", "--config", good_config, "--steps", "10", "--workers", "2", "--out", str(out),
                 "--seed", "1"]) == 0
    assert {"max_eta_L1.txt", "max_speed_L1.txt", "max_inundation_L1.txt", "timing.csv",
            "decomposition.txt"} <= set(os.listdir(out))


@pytest.mark.gpu
def test_duration_flag(cuda_device, good_config, tmp_path, capsys):
    assert main(["run", "--config", good_config, "--duration", "2.0", "--out", str(tmp_path / "d"),
                 "--no-figures"]) == 0
    assert "10 steps" in capsys.readouterr().out


@pytest.mark.gpu
def test_plan_file_roundtrip_and_serial_bytes(cuda_device, good_config, tmp_path):
    out1 = tmp_path / "a"
    assert main(["run", "--config", good_config, "--steps", "6", "--workers", "2", "--out", str(out1),
                 "--no-figures"]) == 0
    out2 = tmp_path / "b"
    assert main(["run", "--config", good_config, "--steps", "6", "--workers", "2", "--decomp",
                 f"file:{out1 / 'decomposition.txt'}", "--out", str(out2), "--no-figures", "--serial"]) == 0
    for name in ("max_eta_L1.txt", "max_speed_L1.txt"):
        assert (out1 / name).read_bytes() == (out2 / name).read_bytes()


@pytest.mark.gpu
def test_snapshots_and_trace(cuda_device, good_config, tmp_path):
    out = tmp_path / "snap"
    assert main(["run", "--config", good_config, "--steps", "6", "--workers", "2", "--snapshot-every", "3",
                 "--out", str(out), "--no-figures"]) == 0
    names = os.listdir(out)
    assert any("step3" in n for n in names) and any("step6" in n for n in names)
    # the snapshot written beside the next chunk holds that step's maxima
    import paper_2408_07609_b200 as P
    from paper_2408_07609_b200 import report as R
    from paper_2408_07609_b200.config import load_config
    system, settings = load_config(good_config)
    sim = P.Simulation(system, settings, P.equal_cell_plan([b.cell_count for _, b in system.all_blocks()], 2))
    sim.run(3, threaded=False)
    R.emit_rasters(system, sim.accumulators, str(tmp_path / "direct"), tag="_step3")
    for f in os.listdir(tmp_path / "direct"):
        assert (out / f).read_bytes() == (tmp_path / "direct" / f).read_bytes(), f
    sim.close()
    trace = tmp_path / "msg.bin"
    assert main(["run", "--config", good_config, "--steps", "2", "--workers", "2", "--trace", str(trace),
                 "--out", str(tmp_path / "tr"), "--no-figures"]) == 0
    assert trace.stat().st_size % 13 == 0 and trace.stat().st_size > 0


@pytest.mark.gpu
def test_worker_abort_flags_partial_outputs(cuda_device, tmp_path):
    """Non-finite bathymetry passes the structural checks and trips the
    numeric guard at the first step: exit 1 and run_failed.txt."""
    np.savetxt(tmp_path / "bad.txt", np.where(np.eye(8, dtype=bool), np.nan, 30.0))
    cfg = tmp_path / "cfg.yaml"
    cfg.write_text("dt: 0.2\nlevels:\n  - dx: 10.0\n    blocks:\n"
                   "      - {origin: [0.0, 0.0], ni: 8, nj: 8, bathymetry: {kind: raster, path: bad.txt}}\n")
    out = tmp_path / "out"
    assert main(["run", "--config", str(cfg), "--steps", "3", "--out", str(out), "--no-figures"]) == 1
    assert "invalid" in (out / "run_failed.txt").read_text()


@pytest.mark.gpu
def test_budgeted_decomposition(cuda_device, tmp_path):
    cfg = tmp_path / "cfg.yaml"
    cfg.write_text(BUDGET_CONFIG)
    out = tmp_path / "out"
    assert main(["run", "--config", str(cfg), "--steps", "4", "--workers", "3", "--out", str(out),
                 "--no-figures"]) == 0
    assert (out / "decomposition.txt").read_text().splitlines()[-1].split() == ["1", "2"]


@pytest.mark.gpu
def test_kochi_trace_per_phase_message_counts(cuda_device, tmp_path):
    """pkg/tests/test_exchange.py:230-260 against the synthesised trace."""
    import paper_2408_07609_b200 as P
    from paper_2408_07609_b200.runner import read_trace
    from paper_2408_07609_b200.schedule import PHASE_ETA
    system = P.build_kochi_scaled_config(0.001)
    fine = system.levels[-1]
    fw = sum(b.ni for b in fine.blocks) * fine.dx
    settings = P.SimulationConfig(dt=0.2, initial=P.InitialCondition(
        "gaussian", 0.3, fw / 8, (fine.blocks[0].origin[0] + fw / 2, fine.blocks[0].origin[1] + 30.0)))
    plan = P.equal_cell_plan([b.cell_count for _, b in system.all_blocks()], 4)
    sim = P.Simulation(system, settings, plan)
    trace = tmp_path / "trace.bin"
    sim.run(2, threaded=True, trace_path=str(trace))
    per_phase = {}
    for (step, code, s, r, ln) in read_trace(str(trace)):
        per_phase[(step, code)] = per_phase.get((step, code), 0) + 1
    eta_expected = sum(1 for (s, r, p) in sim.halo.lengths if p == PHASE_ETA and s != r)
    ig_eta = len({(s, r) for (s, r, p) in sim.tables.pair_links if p == "intergrid-eta" and s != r})
    ig_flux = len({(s, r) for (s, r, p) in sim.tables.pair_links if p == "intergrid-flux" and s != r})
    assert eta_expected and ig_eta and ig_flux
    for step in (0, 1):
        assert per_phase.get((step, 0), 0) == eta_expected
        assert per_phase.get((step, 1), 0) == eta_expected
        assert per_phase.get((step, 2), 0) == ig_eta
        assert per_phase.get((step, 3), 0) == ig_flux
    sim.close()


@pytest.mark.gpu
def test_cli_rasters_equal_a_direct_run(cuda_device, product, tmp_path):
    """`run` on cfg1.yaml: rasters byte-identical to emitting a direct
    Simulation's maxima, plus timing.csv."""
    import systems
    from paper_2408_07609_b200 import report as R
    cfg = os.path.join(os.path.dirname(__file__), "golden", "configs", "cfg1.yaml")
    out = tmp_path / "out"
    assert main(["run", "--config", cfg, "--out", str(out), "--steps", "60"]) == 0
    system, settings, _ = systems.make(product, "cfg1")
    sim = product.Simulation(system, settings)
    sim.run(60, threaded=False)
    R.emit_rasters(system, sim.accumulators, str(tmp_path / "direct"))
    for f in os.listdir(tmp_path / "direct"):
        assert (out / f).read_bytes() == (tmp_path / "direct" / f).read_bytes(), f
    assert (out / "timing.csv").read_text().startswith("rank,steps,mass,momentum")
    sim.close()
