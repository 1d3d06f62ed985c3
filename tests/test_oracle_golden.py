"""Pin the CPU oracle to the reference itself (tests/golden, made by
tests/golden/make_golden.py from the unmodified /root/reference package).

* bitwise: oracle vs the cbrt-aligned reference on every small system, at 1
  and 2 ranks (apply-order semantics), full state incl. ghosts and wet;
* bitwise: oracle vs digests of the cbrt-aligned reference on Kochi-0.001
  (30 steps, 4 ranks), cfg1 (1000 steps) and cfg2 (2000 steps);
* bitwise: single-block kernel calls (mass, momentum, edges, outputs) on
  randomised states with fronts, films and flooded land;
* tolerance (secondary, SURVEY §8(c) ii): oracle vs the stock reference
  (numpy's own np.cbrt);
* the reference's NumericsError message on NaN bathymetry.
"""

import json
import os

import numpy as np
import pytest

import systems
from conftest import GOLDEN

FIELDS = ("eta_old", "eta_new", "m_old", "m_new", "n_old", "n_new")
ACCS = ("max_eta", "max_speed", "max_inundation")


@pytest.fixture(scope="module")
def runs():
    return np.load(os.path.join(GOLDEN, "runs.npz"))


def _eta0(runs, name, system):
    return {b.block_id: runs[f"{name}/eta0/{b.block_id}"] for _, b in system.all_blocks()}


def _plan(P, system, nr):
    return P.equal_cell_plan([b.cell_count for _, b in system.all_blocks()], nr)


@pytest.mark.parametrize("name", systems.SMALL)
@pytest.mark.parametrize("nr", (1, 2))
def test_oracle_bitwise_vs_aligned_reference(oracle_mod, product, runs, name, nr):
    system, settings, n = systems.make(product, name)
    if nr > system.n_blocks:
        pytest.skip("single block")
    sim = oracle_mod.OracleSimulation(system, settings, _plan(product, system, nr),
                                      eta0=_eta0(runs, name, system))
    sim.run(n)
    for bid, st in sim.states.items():
        pre = f"{name}/{nr}/aligned/{bid}"
        for f in FIELDS:
            assert np.array_equal(getattr(st, f), runs[f"{pre}/{f}"]), (bid, f)
        assert np.array_equal(st.wet.astype(bool), runs[f"{pre}/wet"]), (bid, "wet")
        for f in ACCS:
            assert np.array_equal(getattr(st, f), runs[f"{pre}/{f}"]), (bid, f)


@pytest.mark.parametrize("name", systems.SMALL)
def test_oracle_vs_stock_reference_tolerance(oracle_mod, product, runs, name):
    """Secondary: against numpy's own cbrt the scheme is discontinuous, so
    differences may grow past ulp level; bound them relative to the field."""
    system, settings, n = systems.make(product, name)
    sim = oracle_mod.OracleSimulation(system, settings, eta0=_eta0(runs, name, system))
    sim.run(n)
    for bid, st in sim.states.items():
        pre = f"{name}/1/stock/{bid}"
        for f in ("eta_old", "m_old", "n_old") + ACCS:
            ref = runs[f"{pre}/{f}"]
            got = getattr(st, f)
            scale = max(1e-12, float(np.max(np.abs(ref))))
            assert np.max(np.abs(got - ref)) <= 1e-3 * scale, (bid, f)
        # wet/dry mask identical except within 1e-9 m of the threshold
        d = st.h_ext + st.eta_new
        w_ref = runs[f"{pre}/wet"]
        near = np.abs(d - settings.wet_threshold) < 1e-9
        assert np.array_equal(st.wet.astype(bool)[~near], w_ref[~near])


@pytest.fixture(scope="module")
def digests():
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ("kochi", "cfg1", "cfg2"))
def test_oracle_bitwise_vs_reference_digests(oracle_mod, product, digests, name):
    d = digests[name]
    system, settings, n = systems.make(product, name)
    eta0 = systems.eta0_of(system, settings)
    if any(systems.digest(eta0[b.block_id]) != d["eta0"][str(b.block_id)] for _, b in system.all_blocks()) \
            or any(systems.digest(b.h) != d["h"][str(b.block_id)] for _, b in system.all_blocks()):
        pytest.skip("this host's libm (np.exp / np.power) differs from the golden host's")
    sim = oracle_mod.OracleSimulation(system, settings, _plan(product, system, d["ranks"]))
    sim.run(n)
    for bid, st in sim.states.items():
        for f in FIELDS + ACCS:
            assert systems.digest(getattr(st, f)) == d["aligned"][f"{bid}/{f}"], (bid, f)


@pytest.mark.parametrize("name,tol_eta,tol_acc", (("cfg1", 1e-13, 1e-13), ("cfg2", 3e-3, 3e-3)))
def test_oracle_vs_stock_reference_big(oracle_mod, product, name, tol_eta, tol_acc):
    """cfg1 stays ulp-level; cfg2's wet/dry fronts amplify 1-ulp cbrt
    differences to ~1e-4 m (SURVEY §8(c) noise floors)."""
    system, settings, n = systems.make(product, name)
    ref = np.load(os.path.join(GOLDEN, f"{name}_stock.npz"))
    sim = oracle_mod.OracleSimulation(system, settings)
    sim.run(n)
    for bid, st in sim.states.items():
        got = st.interior(st.eta_old)
        r = ref[f"{bid}/eta_old"].astype(float)
        assert np.max(np.abs(got - r)) <= tol_eta * max(1.0, np.max(np.abs(r)))
        for f in ("max_eta", "max_inundation"):
            r = ref[f"{bid}/{f}"].astype(float)
            assert np.max(np.abs(getattr(st, f) - r)) <= tol_acc * max(1.0, np.max(np.abs(r)))


@pytest.mark.parametrize("case", ("scalar", "percell"))
def test_oracle_kernels_bitwise(oracle_mod, product, case):
    k = np.load(os.path.join(GOLDEN, "kernels.npz"))
    h, eta0 = k[f"{case}/in_h"], k[f"{case}/in_eta0"]
    nman = k[f"{case}/in_nman"]
    ni, nj = h.shape
    blk = product.Block(1, (0.0, 0.0), ni, nj, h, float(nman) if nman.ndim == 0 else nman)
    sim = oracle_mod.single_block_sim(blk, 10.0, product.SimulationConfig(dt=0.2), eta0=eta0)
    st = sim.states[1]
    st.m_old[...] = k[f"{case}/in_m0"]
    st.n_old[...] = k[f"{case}/in_n0"]
    sim.phase("mass")
    assert np.array_equal(st.eta_new, k[f"{case}/mass_eta_new"])
    assert np.array_equal(st.wet.astype(bool), k[f"{case}/mass_wet"])
    sim.phase("momentum")
    assert np.array_equal(st.m_new, k[f"{case}/mom_m_new"])
    assert np.array_equal(st.n_new, k[f"{case}/mom_n_new"])
    lib = oracle_mod.lib()
    import ctypes
    for side, kind, iv in ((0, 1, (1, 7)), (1, 0, (0, nj)), (2, 1, (0, ni)), (3, 1, (2, 11))):
        lib.oracle_edge(ctypes.byref(sim.blocks[0]), ctypes.c_int64(sim.sim.cur), ctypes.c_int64(side),
                        ctypes.c_int64(kind), ctypes.c_int64(iv[0]), ctypes.c_int64(iv[1]))
    assert np.array_equal(st.m_new, k[f"{case}/edge_m_new"])
    assert np.array_equal(st.n_new, k[f"{case}/edge_n_new"])
    sim.phase("output")
    sim.phase("output")
    for f in ACCS:
        assert np.array_equal(getattr(st, f), k[f"{case}/acc_{f}"]), f


def test_oracle_error_message(oracle_mod, product):
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        want = json.load(f)["nan_bathymetry"]
    T = product
    system = T.NestedGridSystem(levels=[T.GridLevel(1, 10.0, [
        systems.flat_block(T, 1, (0.0, 0.0), 8, 8, 30.0),
        T.Block(2, (80.0, 0.0), 8, 8, np.where(np.eye(8, dtype=bool), np.nan, 30.0))])])
    sim = oracle_mod.OracleSimulation(system, T.SimulationConfig(dt=0.2))
    with pytest.raises(oracle_mod.OracleNumericsError) as ei:
        sim.run(3)
    assert str(ei.value) == want


def test_oracle_error_message_dry_basin_threshold0(oracle_mod, product):
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        want = json.load(f)["dry_basin_threshold0"]
    T = product
    system = T.NestedGridSystem(levels=[T.GridLevel(1, 10.0, [
        T.Block(1, (0.0, 0.0), 6, 5, np.zeros((6, 5)))])])
    sim = oracle_mod.OracleSimulation(system, T.SimulationConfig(dt=0.1, wet_threshold=0.0))
    with pytest.raises(oracle_mod.OracleNumericsError) as ei:
        sim.run(3)
    assert str(ei.value) == want


def test_oracle_kochi6h_first_checkpoint(oracle_mod, product):
    """The 6-hour golden's first checkpoint (1000 steps of Kochi-0.001 on the
    cbrt-aligned reference); the full 37,000-step run and the reference's
    blow-up are checked against the product on the GPU, and against the
    oracle with TSUNAMI_SLOW=1."""
    with open(os.path.join(GOLDEN, "kochi6h.json")) as f:
        g = json.load(f)
    system, settings, _ = systems.kochi(product, 0.001)
    eta0 = systems.eta0_of(system, settings)
    if any(systems.digest(eta0[b.block_id]) != g["eta0"][str(b.block_id)] for _, b in system.all_blocks()):
        pytest.skip("this host's libm (np.exp) differs from the golden host's")
    sim = oracle_mod.OracleSimulation(system, settings)
    targets = sorted(int(k) for k in g["checkpoints"])
    if os.environ.get("TSUNAMI_SLOW") != "1":
        targets = targets[:1]
    done = 0
    for target in targets:
        sim.run(target - done)
        done = target
        want = g["checkpoints"][str(target)]
        for bid, st in sim.states.items():
            for f in ("eta_old", "m_old", "n_old") + ACCS:
                assert systems.digest(getattr(st, f)) == want[f"{bid}/{f}"], (target, bid, f)
    if os.environ.get("TSUNAMI_SLOW") == "1":
        with pytest.raises(oracle_mod.OracleNumericsError) as ei:
            sim.run(g["failure"]["within"])
        assert str(ei.value) == g["failure"]["message"]
