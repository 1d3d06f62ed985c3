"""The reference's run-level contract on the GPU path (tests/test_runner.py,
tests/test_acceptance.py of the reference, ported to the product API)."""

import json
import os

import numpy as np
import pytest

import systems
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _plan(P, system, nr):
    return P.equal_cell_plan([b.cell_count for _, b in system.all_blocks()], nr)


def _nan_system(T):
    return T.NestedGridSystem(levels=[T.GridLevel(1, 10.0, [
        systems.flat_block(T, 1, (0.0, 0.0), 8, 8, 30.0),
        T.Block(2, (80.0, 0.0), 8, 8, np.where(np.eye(8, dtype=bool), np.nan, 30.0))])])


def test_numerics_error_message_matches_reference(cuda_device, product):
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        want = json.load(f)["nan_bathymetry"]
    system = _nan_system(product)
    sim = product.Simulation(system, product.SimulationConfig(dt=0.2), _plan(product, system, 1))
    with pytest.raises(product.NumericsError) as ei:
        sim.run(3, threaded=False)
    assert str(ei.value) == want


def test_numerics_error_dry_basin_threshold0(cuda_device, product):
    """wet_threshold 0 over a dry basin: the reference's all-wet branch
    divides 0/0 and raises NumericsError (golden made by the reference)."""
    with open(os.path.join(GOLDEN, "errors.json")) as f:
        want = json.load(f)["dry_basin_threshold0"]
    T = product
    system = T.NestedGridSystem(levels=[T.GridLevel(1, 10.0, [
        T.Block(1, (0.0, 0.0), 6, 5, np.zeros((6, 5)))])])
    sim = T.Simulation(system, T.SimulationConfig(dt=0.1, wet_threshold=0.0), _plan(T, system, 1))
    with pytest.raises(T.NumericsError) as ei:
        sim.run(3, threaded=False)
    assert str(ei.value) == want


def test_worker_failure_aborts_threaded_run(cuda_device, product):
    """tests/test_runner.py:102-112: multi-rank runs wrap it in SimulationAborted."""
    system = _nan_system(product)
    sim = product.Simulation(system, product.SimulationConfig(dt=0.2), _plan(product, system, 2))
    with pytest.raises(product.SimulationAborted):
        sim.run(3, threaded=True, timeout=5.0)


def test_lake_at_rest_bitwise(cuda_device, product):
    """tests/test_acceptance.py:60-81 (trench, land, island, sub-threshold film)."""
    n = 150
    h = np.full((n, n), 30.0)
    h[:, :20] = 95.0
    h[120:, :] = -5.0
    h[40:55, 60:75] = -2.0
    h[60:80, 80:100] = 0.5e-5
    T = product
    system = T.NestedGridSystem(levels=[T.GridLevel(1, 10.0, [T.Block(1, (0.0, 0.0), n, n, h)])])
    sim = T.Simulation(system, T.SimulationConfig(dt=0.2), _plan(T, system, 1))
    sim.run(1000, threaded=False)
    st = sim.states[1]
    assert np.max(np.abs(st.interior(st.eta_old))) == 0.0
    assert np.all(st.m_old == 0.0) and np.all(st.n_old == 0.0)


def test_mass_conservation_closed_basin(cuda_device, product):
    """tests/test_acceptance.py:84-102."""
    n, dx = 120, 10.0
    T = product
    system = T.NestedGridSystem(levels=[T.GridLevel(1, dx, [systems.flat_block(T, 1, (0.0, 0.0), n, n, 50.0)])])
    sim = T.Simulation(system, systems.hump(T, 1.0, 80.0, (600.0, 600.0)), _plan(T, system, 1))
    st = sim.states[1]
    vol0 = float(np.sum(st.interior(st.eta_old))) * dx * dx
    water0 = float(np.sum(50.0 + st.interior(st.eta_old))) * dx * dx
    sim.run(1000, threaded=False)
    vol1 = float(np.sum(st.interior(st.eta_old))) * dx * dx
    assert abs(vol1 - vol0) / water0 < 1e-10


def test_mirror_symmetry_with_on_step(cuda_device, product):
    """tests/test_acceptance.py:105-131 through the serial on_step hook."""
    n, dx = 60, 10.0
    h = np.empty((n, n))
    h[:] = 30.0 - 0.3 * (np.arange(n) + 0.5)[None, :]
    h[28:32, 10:14] = -2.0
    T = product
    system = T.NestedGridSystem(levels=[T.GridLevel(1, dx, [T.Block(1, (0.0, 0.0), n, n, h)])])
    sim = T.Simulation(system, systems.hump(T, 0.8, 80.0, (300.0, 200.0)), _plan(T, system, 1))
    worst = [0.0]

    def check(s, step):
        st = s.states[1]
        g = st.halo
        e = st.interior(st.eta_old)
        a = float(np.max(np.abs(e - e[::-1, :])))
        m = st.m_old[g:g + n + 1, g:g + n]
        a = max(a, float(np.max(np.abs(m + m[::-1, :]))))
        nn = st.n_old[g:g + n, g:g + n + 1]
        a = max(a, float(np.max(np.abs(nn - nn[::-1, :]))))
        worst[0] = max(worst[0], a)

    sim.run(500, threaded=False, on_step=check)
    assert worst[0] < 1e-12
    with pytest.raises(ValueError):
        sim.run(1, threaded=True, on_step=check)


def test_nested_matches_uniform_fine(cuda_device, product):
    """tests/test_acceptance.py:265-290."""
    T = product
    settings = systems.hump(T, 0.2, 60.0, (240.0, 360.0), dt=0.1)
    fine = T.NestedGridSystem(levels=[T.GridLevel(1, 3.0, [systems.flat_block(T, 1, (0.0, 0.0), 240, 240, 5.0)])])
    nested = T.NestedGridSystem(levels=[
        T.GridLevel(1, 9.0, [systems.flat_block(T, 1, (0.0, 0.0), 80, 80, 5.0)]),
        T.GridLevel(2, 3.0, [systems.flat_block(T, 2, (180.0, 180.0), 120, 120, 5.0)])])
    sf = T.Simulation(fine, settings, _plan(T, fine, 1))
    sn = T.Simulation(nested, settings, _plan(T, nested, 1))
    worst = 0.0
    for _ in range(200):
        sf.run(1, threaded=False)
        sn.run(1, threaded=False)
        ef = sf.states[1].interior(sf.states[1].eta_old)[60:180, 60:180]
        en = sn.states[2].interior(sn.states[2].eta_old)
        worst = max(worst, float(np.sqrt(np.mean((ef - en) ** 2))))
    assert worst / 0.2 <= 0.05


def test_zero_steps_and_report(cuda_device, product):
    system, settings, _ = systems.chain(product)
    sim = product.Simulation(system, settings, _plan(product, system, 2))
    rep = sim.run(0, threaded=False)
    assert rep.steps == 0
    for acc in sim.accumulators.values():
        assert np.all(acc.max_eta == 0.0) and np.all(acc.max_speed == 0.0)
    rep = sim.run(5, threaded=True, record_phases=True)
    assert rep.n_ranks == 2
    for rt in rep.ranks:
        assert set(rt.routines) == set(product.ROUTINES)
        assert all(v >= 0.0 for v in rt.routines.values())
        assert rt.total >= sum(rt.routines.values()) * 0.5
    for ctx in sim.contexts:
        assert ctx.phase_log == list(product.PHASE_SEQUENCE) * 5
    # seam propagation (tests/test_runner.py:92-98)
    sim.run(55, threaded=True)
    assert sim.accumulators[3].max_eta.max() > 1e-4


def test_message_trace(cuda_device, product, tmp_path):
    from paper_2408_07609_b200.runner import read_trace
    system, settings, _ = systems.kochi(product)
    sim = product.Simulation(system, settings, _plan(product, system, 4))
    path = str(tmp_path / "trace.bin")
    sim.run(3, trace_path=path)
    recs = read_trace(path)
    assert recs and all(r[2] != r[3] for r in recs)
    assert sorted({r[0] for r in recs}) == [0, 1, 2]
    assert {r[1] for r in recs} <= {0, 1, 2, 3}


def test_end_to_end_host_buffers_match_fresh_run(cuda_device, product):
    """The e2e leg of bench.py: reset of a used simulation + batched upload
    of page-locked inputs + run + batched download into page-locked buffers
    gives exactly a fresh simulation's state."""
    from paper_2408_07609_b200.runner import host_block_arrays
    system, settings, _ = systems.make(product, "quad_wetdry")
    plan = _plan(product, system, 1)
    fresh = product.Simulation(system, settings, plan)
    fresh.run(25, threaded=False)
    sim = product.Simulation(system, settings, plan)
    sim.run(7, threaded=False)                 # a used state: fluxes, maxima, step count
    sim.reset()
    arrays = host_block_arrays(system, settings, pinned=True)
    nbytes = sim.upload_initial_state(arrays)
    assert nbytes == sum(a[0].nbytes + a[2].nbytes for a in arrays.values())
    sim.run(25, threaded=False)
    outs = sim.output_buffers(pinned=True)
    got, nb = sim.download_outputs(outs)
    assert nb == sum(a.nbytes for bufs in outs.values() for a in bufs)
    for bid, (me, ms, mi, eo) in got.items():
        acc = fresh.accumulators[bid]
        assert np.array_equal(me, acc.max_eta)
        assert np.array_equal(ms, acc.max_speed)
        assert np.array_equal(mi, acc.max_inundation)
        assert np.array_equal(eo, fresh.states[bid].eta_old)
        for f in ("eta_new", "m_old", "m_new", "n_old", "n_new"):
            assert np.array_equal(getattr(sim.states[bid], f), getattr(fresh.states[bid], f)), f


def test_cost_model_measured_fitted_saved_loaded_and_planned(cuda_device, product, tmp_path):
    """(f)2: the B200 replacement of measure_momentum_cost (balance.py:301-328)
    measures per-block step costs on the device, fit_cost_model fits them,
    the reference's model file round-trips, and the plans use it; the
    per-width table feeds packed_plan."""
    P = product
    samples = P.measure_block_costs([6000, 60000, 600000], repeats=2, steps=5, min_cells=2e6)
    assert [c for c, _ in samples] == [6000, 60000, 600000] and all(t > 0 for _, t in samples)
    assert samples[2][1] > samples[0][1]
    model = P.fit_cost_model(samples)
    assert model.slope > 0 and model.r_squared > 0.9
    path = str(tmp_path / "model.txt")
    P.save_cost_model(model, path)
    back = P.load_cost_model(path)
    assert back == model
    system = P.build_kochi_scaled_config(0.01)
    cells = [b.cell_count for _, b in system.all_blocks()]
    plan = P.minmax_plan(cells, 4, back)
    assert plan.n_ranks == 4 and P.rank_costs(plan, back).max() <= P.rank_costs(P.equal_cell_plan(cells, 4),
                                                                                back).max() + 1e-9
    table = P.measure_width_costs((36, 60), cells=4e6, steps=5)
    assert set(table) == {36, 60} and all(v["step_ps_per_cell"] > 0 for v in table.values())
    P.save_width_costs(table, str(tmp_path / "w.json"))
    packed = P.packed_plan(system, 4, table=P.load_width_costs(str(tmp_path / "w.json")))
    assert packed.n_ranks == 4 and sorted(set(packed.owners)) == [0, 1, 2, 3]


@pytest.mark.parametrize("name", ("kochi", "cfg5"))
def test_device_built_bathymetry_equals_host_setup(cuda_device, product, name):
    """(f)3: blocks whose depth is a 1-D profile get h_ext built on the
    device (edge replication + the siblings' strips), bit-identical to the
    host setup (kernels.py:108-112, exchange.py:281-300)."""
    from paper_2408_07609_b200.runner import h_profile, host_block_arrays
    system, settings, _ = systems.kochi(product, 0.001) if name == "kochi" else systems.cfg5(product, 0.02)
    assert all(h_profile(b) is not None for _, b in system.all_blocks())
    host = host_block_arrays(system, settings)
    sim = product.Simulation(system, settings)
    for bid, st in sim.states.items():
        assert np.array_equal(st.h_ext.view(np.uint64), host[bid][0].view(np.uint64)), bid
    sim.close()


def test_end_to_end_with_device_bathymetry(cuda_device, product):
    """The e2e leg on a system with 1-D depth profiles (Kochi): the profiles
    are uploaded and expanded on the device instead of ghosted h_ext;
    the result equals a fresh run."""
    from paper_2408_07609_b200.runner import host_block_arrays
    system, settings, _ = systems.kochi(product, 0.001)
    fresh = product.Simulation(system, settings)
    fresh.run(12, threaded=False)
    sim = product.Simulation(system, settings)
    sim.run(5, threaded=False)
    sim.reset()
    arrays = host_block_arrays(system, settings, pinned=True, device_bathymetry=True)
    assert all(a[0] is None for a in arrays.values())
    nbytes = sim.upload_initial_state(arrays)
    assert nbytes < sum(a[2].nbytes for a in arrays.values()) * 1.1
    sim.run(12, threaded=False)
    outs = sim.output_buffers(pinned=True, fields=sim.RESULT_FIELDS)
    got, _ = sim.download_outputs(outs)
    for bid, maps in got.items():
        for f, m in zip(sim.RESULT_FIELDS, maps):
            assert np.array_equal(m.view(np.uint64), getattr(fresh.accumulators[bid], f).view(np.uint64)), (bid, f)
        for f in ("eta_old", "m_old", "n_old", "h_ext"):
            a, b = getattr(sim.states[bid], f), getattr(fresh.states[bid], f)
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64)), (bid, f)
    sim.close()
    fresh.close()


def test_edited_bathymetry_of_a_profiled_block(cuda_device, oracle_mod, product):
    """The mass kernel reads a profiled block's depth from its 1-D profile;
    an in-place edit of h_ext (kernels.py BlockState arrays are writable)
    must replace it: the run equals the oracle's on the edited depth."""
    system, settings, _ = systems.kochi(product, 0.001)
    plan = _plan(product, system, 1)
    gpu = product.Simulation(system, settings, plan)
    orc = oracle_mod.OracleSimulation(system, settings, plan)
    gpu.run(3, threaded=False)
    orc.run(3)
    bid = system.all_blocks()[-1][1].block_id
    for st in (gpu.states[bid], orc.states[bid]):
        st.h_ext[4, 5] += 7.25
        st.h_ext[6, 3] *= 0.5
    gpu.run(6, threaded=False)
    orc.run(6)
    for b, o in orc.states.items():
        g = gpu.states[b]
        for f in ("eta_old", "m_old", "n_old", "h_ext"):
            assert np.array_equal(getattr(g, f).view(np.uint64), getattr(o, f).view(np.uint64)), (b, f)
        for f in ("max_eta", "max_speed", "max_inundation"):
            a, c = getattr(gpu.accumulators[b], f), getattr(o, f)
            assert np.array_equal(a.view(np.uint64), np.asarray(c).view(np.uint64)), (b, f)
    gpu.close()


def test_trace_step_is_a_step(cuda_device, product):
    """ts_trace_step (tools/trace_step.py) advances the state exactly as
    ts_run(1) does, and reports every launch of the step."""
    import ctypes
    from paper_2408_07609_b200 import _native as N
    system, settings, _ = systems.kochi(product, 0.001)
    plan = _plan(product, system, 1)
    a = product.Simulation(system, settings, plan)
    a.run(2, threaded=False)
    a.run(1, threaded=False)
    a.run(2, threaded=False)
    b = product.Simulation(system, settings, plan)
    b.run(2, threaded=False)
    lab, us, cnt = (ctypes.c_int32 * 64)(), (ctypes.c_float * 64)(), ctypes.c_int32()
    N.check(N.lib().ts_trace_step(b._h, lab, us, 64, ctypes.byref(cnt)))
    b._invalidate()
    b.steps_done += 1
    b.run(2, threaded=False)
    assert cnt.value == b.launches_per_step
    assert all(us[k] >= 0.0 for k in range(cnt.value))
    for bid in a.states:
        for f in ("eta_old", "m_old", "n_old"):
            assert np.array_equal(getattr(a.states[bid], f).view(np.uint64),
                                  getattr(b.states[bid], f).view(np.uint64)), (bid, f)
        for f in ("max_eta", "max_speed", "max_inundation"):
            assert np.array_equal(getattr(a.accumulators[bid], f).view(np.uint64),
                                  getattr(b.accumulators[bid], f).view(np.uint64)), (bid, f)
    a.close()
    b.close()
