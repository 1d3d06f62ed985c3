"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

The gate is bitwise equality (==, NaN-aware) of every array the reference
exposes — eta/M/N in both buffer roles including ghost rings, the derived
wet mask against the oracle's stored one, and the three running maxima —
after full runs of every fixture system, at 1 and 2 ranks, split across
several ``run`` calls (re-entrancy), on BASELINE configs 1 and 2 at their
full step counts, on the Kochi-shaped 5-level domain at scale 0.001 and a
short window at the full 47 M-cell scale.  Phase-level and kernel-level
parity pin each kernel separately.
"""

import numpy as np
import pytest

import systems

pytestmark = pytest.mark.gpu

FIELDS = ("eta_old", "eta_new", "m_old", "m_new", "n_old", "n_new")
ACCS = ("max_eta", "max_speed", "max_inundation")


def _plan(P, system, nr):
    return P.equal_cell_plan([b.cell_count for _, b in system.all_blocks()], nr)


def _same_bits(a, b):
    """Elementwise identical IEEE bit patterns (so -0.0 != +0.0); any NaN
    equals any NaN (payloads of a failed step are not compared)."""
    a, b = np.ascontiguousarray(a, dtype=np.float64), np.ascontiguousarray(b, dtype=np.float64)
    return (a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))


def bits_equal(a, b):
    return np.shape(a) == np.shape(b) and bool(np.all(_same_bits(a, b)))


def assert_same(gpu, orc, where="", wet="all"):
    """``wet="interior"`` between mass and halo-eta: the reference refreshes
    ghost wet flags only when halo-eta writes the ghosts, so until then they
    describe the previous step (never read in that window)."""
    for bid, o in orc.states.items():
        g = gpu.states[bid]
        for f in FIELDS:
            a, b = getattr(g, f), getattr(o, f)
            if not bits_equal(a, b):
                bad = np.argwhere(~_same_bits(a, b))
                raise AssertionError(f"{where} block {bid} {f}: {len(bad)} cells differ, first "
                                     f"{bad[0].tolist()} gpu={a[tuple(bad[0])]!r} "
                                     f"oracle={b[tuple(bad[0])]!r}")
        gw, ow = g.wet, o.wet.astype(bool)
        if wet == "interior":
            gw, ow = g.interior(gw), o.interior(ow)
        assert np.array_equal(gw, ow), (where, bid, "wet")
        acc = gpu.accumulators[bid]
        for f in ACCS:
            assert bits_equal(getattr(acc, f), getattr(o, f)), (where, bid, f)


@pytest.mark.parametrize("name", systems.SMALL + ("kochi",))
@pytest.mark.parametrize("nr", (1, 2))
def test_run_parity(cuda_device, oracle_mod, product, name, nr):
    system, settings, n = systems.make(product, name)
    if nr > system.n_blocks:
        pytest.skip("single block")
    plan = _plan(product, system, nr)
    gpu = product.Simulation(system, settings, plan)
    orc = oracle_mod.OracleSimulation(system, settings, plan)
    assert_same(gpu, orc, "initial")
    done = 0
    for chunk in (1, 2, n // 3, n - 3 - n // 3):
        gpu.run(chunk, threaded=False)
        orc.run(chunk)
        done += chunk
        assert_same(gpu, orc, f"after {done} steps")
    gpu.close()


@pytest.mark.parametrize("name", ("quad_wetdry", "chain", "kochi"))
def test_per_stage_exchange_path(cuda_device, oracle_mod, product, name, monkeypatch):
    """TSUNAMI_B200_MERGED=0: every exchange stage as its own launch (the
    path ts_phase uses) is bitwise the oracle as well."""
    monkeypatch.setenv("TSUNAMI_B200_MERGED", "0")
    system, settings, n = systems.make(product, name)
    plan = _plan(product, system, 2 if system.n_blocks > 1 else 1)
    gpu = product.Simulation(system, settings, plan)
    orc = oracle_mod.OracleSimulation(system, settings, plan)
    gpu.run(n, threaded=False)
    orc.run(n)
    assert_same(gpu, orc, f"per-stage path after {n} steps")
    gpu.close()


def test_merged_exchange_is_the_default(cuda_device, product, monkeypatch):
    """Kochi at one GPU: mass, at most four march launches and at most two
    launches per exchange phase (its writes, then the second-wave writes
    whose destinations the phase also reads); the per-stage path has more."""
    system, settings, _ = systems.make(product, "kochi")
    plan = _plan(product, system, 1)
    monkeypatch.delenv("TSUNAMI_B200_MERGED", raising=False)
    merged = product.Simulation(system, settings, plan)
    merged.run(1, threaded=False)
    monkeypatch.setenv("TSUNAMI_B200_MERGED", "0")
    staged = product.Simulation(system, settings, plan)
    staged.run(1, threaded=False)
    assert merged.launches_per_step <= 1 + 4 + 2 * 2
    assert merged.launches_per_step < staged.launches_per_step
    merged.close()
    staged.close()


def test_cfg5_quarter_scale_window(cuda_device, oracle_mod, product):
    """BASELINE config 5 at 1/4 of its cells (10,000 x 10,000 = 100 M cells
    in 8 strips of 1250 x 10,000), 6 steps, bitwise."""
    system, settings, _ = systems.cfg5(product, 0.5)
    assert system.cell_count == 100_000_000
    plan = _plan(product, system, 1)
    gpu = product.Simulation(system, settings, plan)
    orc = oracle_mod.OracleSimulation(system, settings, plan)
    for chunk in (1, 5):
        gpu.run(chunk, threaded=False)
        orc.run(chunk)
    assert_same(gpu, orc, "cfg5 quarter scale")
    gpu.close()


@pytest.mark.parametrize("nr", (1, 4))
def test_cfg5_strips_parity(cuda_device, oracle_mod, product, nr):
    """BASELINE config 5 (single 10 m level in 8 abutting strips, coast in
    the last strip) at 1/50 scale: 400 x 400 cells, 200 steps."""
    system, settings, n = systems.cfg5(product, 0.02)
    plan = _plan(product, system, nr)
    gpu = product.Simulation(system, settings, plan)
    orc = oracle_mod.OracleSimulation(system, settings, plan)
    gpu.run(n, threaded=False)
    orc.run(n)
    assert_same(gpu, orc, f"cfg5 after {n} steps")
    gpu.close()


@pytest.mark.parametrize("name", ("cfg1", "cfg2"))
def test_baseline_config_parity(cuda_device, oracle_mod, product, name):
    """BASELINE configs 1 and 2 at their full step counts (1000 / 2000)."""
    system, settings, n = systems.make(product, name)
    gpu = product.Simulation(system, settings)
    orc = oracle_mod.OracleSimulation(system, settings)
    gpu.run(n, threaded=False)
    orc.run(n)
    assert_same(gpu, orc, name)
    land = sum(int(np.count_nonzero(gpu.accumulators[b].max_inundation)) for b in gpu.states)
    assert land > 0                       # the wet/dry front moved inland


def test_kochi_full_scale_window(cuda_device, oracle_mod, product):
    """The 47,211,444-cell 5-level domain (BASELINE config 3): a 103-step
    window (SURVEY.md:313), bitwise, with the 4-rank plan's apply order;
    compared after the first step, after 3 and at the end."""
    system, settings, _ = systems.kochi(product, 1.0)
    plan = _plan(product, system, 4)
    gpu = product.Simulation(system, settings, plan)
    orc = oracle_mod.OracleSimulation(system, settings, plan)
    done = 0
    for chunk in (1, 2, 100):
        gpu.run(chunk, threaded=False)
        orc.run(chunk)
        done += chunk
        if chunk != 2:
            assert_same(gpu, orc, f"kochi-1.0 after {done} steps")
    gpu.close()


GPU_PHASES = {"momentum": ("momentum", "edges")}


@pytest.mark.parametrize("name", ("identity3", "quad_wetdry"))
def test_phase_parity(cuda_device, oracle_mod, product, name):
    """Each phase of runner.PHASE_SEQUENCE separately (gather-then-scatter
    hazards in identity3; ragged halos and fronts in quad_wetdry)."""
    system, settings, _ = systems.make(product, name)
    gpu = product.Simulation(system, settings)
    orc = oracle_mod.OracleSimulation(system, settings)
    for step in range(6):
        for ph in ("mass", "restrict", "halo-eta", "momentum", "prolong", "halo-flux", "output", "swap"):
            orc.phase(ph)
            for gph in GPU_PHASES.get(ph, (ph,)):
                gpu.phase(gph)
            assert_same(gpu, orc, f"step {step} {ph}",
                        wet="interior" if ph in ("mass", "restrict") else "all")


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("per_cell", (False, True))
def test_kernel_parity_random_states(cuda_device, oracle_mod, product, seed, per_cell):
    """update_mass / update_momentum / accumulate on randomised states with
    land, sub-threshold films, fronts and random ghost fluxes
    (cf. tests/test_kernels.py:395-419)."""
    rng = np.random.default_rng(100 + seed)
    ni, nj = int(rng.integers(5, 70)), int(rng.integers(3, 140))
    h = rng.uniform(-1.0, 6.0, (ni, nj))
    h[rng.random((ni, nj)) < 0.15] = 2e-6
    nman = 0.01 + 0.05 * rng.random((ni, nj)) if per_cell else 0.03
    blk = product.Block(1, (0.0, 0.0), ni, nj, h, nman)
    eta0 = np.where(h > 0, rng.normal(0.0, 0.3, (ni, nj)), 0.0)
    settings = product.SimulationConfig(dt=0.2)
    system = product.NestedGridSystem(levels=[product.GridLevel(1, 10.0, [blk])])
    gpu = product.Simulation(system, settings)
    orc = oracle_mod.single_block_sim(blk, 10.0, settings)
    m0 = rng.normal(0.0, 0.4, (ni + 5, nj + 4))
    n0 = rng.normal(0.0, 0.4, (ni + 4, nj + 5))
    for sim in (gpu, orc):
        st = sim.states[1]
        st.eta_old[2:-2, 2:-2] = eta0
        st.eta_new[2:-2, 2:-2] = eta0
        st.m_old[...] = m0
        st.n_old[...] = n0
    orc.states[1].refresh_wet(settings.wet_threshold)
    for ph in ("mass", "momentum", "output", "output"):
        orc.phase(ph)
        gpu.phase(ph)
        assert_same(gpu, orc, ph)


def test_device_cbrt_bitwise(cuda_device, oracle_mod):
    from paper_2408_07609_b200 import _native
    rng = np.random.default_rng(5)
    x = np.concatenate([np.exp(rng.uniform(np.log(1e-8), np.log(1e6), 2_000_000)),
                        2.0 ** np.arange(-60, 60.0), [0.0, -0.0, np.inf, -8.0, 5e-324, 1e-310]])
    d = _native.cbrt_device(x)
    assert np.array_equal(d.view(np.uint64), _native.cbrt_host(x).view(np.uint64))
    assert np.array_equal(d.view(np.uint64), oracle_mod.cbrt(x).view(np.uint64))


@pytest.mark.parametrize("scale", (1e-300, 5e-320, 1e120))
def test_kernel_parity_extreme_magnitudes(cuda_device, oracle_mod, product, scale):
    """Fluxes near the exponent limits (tiny, subnormal, huge) take the
    exact-arithmetic re-run of the momentum tiles (fastmath.cuh guards);
    results stay bitwise equal to the oracle."""
    rng = np.random.default_rng(7)
    ni, nj = 40, 30
    h = rng.uniform(0.5, 6.0, (ni, nj))
    blk = product.Block(1, (0.0, 0.0), ni, nj, h, 0.03)
    settings = product.SimulationConfig(dt=0.2)
    system = product.NestedGridSystem(levels=[product.GridLevel(1, 10.0, [blk])])
    gpu = product.Simulation(system, settings)
    orc = oracle_mod.single_block_sim(blk, 10.0, settings)
    m0 = rng.normal(0.0, 1.0, (ni + 5, nj + 4))
    n0 = rng.normal(0.0, 1.0, (ni + 4, nj + 5))
    m0[10:20, :] *= scale
    n0[:, 5:9] *= scale
    for sim in (gpu, orc):
        sim.states[1].m_old[...] = m0
        sim.states[1].n_old[...] = n0
    for ph in ("mass", "momentum", "output"):
        orc.phase(ph)
        gpu.phase(ph)
        assert_same(gpu, orc, ph)


def test_kochi_six_hours_vs_reference_golden(cuda_device, product):
    """The 6-hour golden (tests/golden/make_golden_6h.py): the cbrt-aligned
    reference on Kochi-0.001, digests at 1000 / 10000 / 36000 / 37000 steps,
    then the reference's own blow-up inside the next 1000 steps with its
    NumericsError message.  The product must reproduce all of it."""
    import json
    import os
    from conftest import GOLDEN
    with open(os.path.join(GOLDEN, "kochi6h.json")) as f:
        g = json.load(f)
    system, settings, _ = systems.kochi(product, 0.001)
    eta0 = systems.eta0_of(system, settings)
    if any(systems.digest(eta0[b.block_id]) != g["eta0"][str(b.block_id)] for _, b in system.all_blocks()):
        pytest.skip("this host's libm (np.exp) differs from the golden host's")
    sim = product.Simulation(system, settings, _plan(product, system, 1))
    done = 0
    for target in sorted(int(k) for k in g["checkpoints"]):
        sim.run(target - done, threaded=False)
        done = target
        want = g["checkpoints"][str(target)]
        for bid, st in sim.states.items():
            for f in ("eta_old", "m_old", "n_old"):
                assert systems.digest(getattr(st, f)) == want[f"{bid}/{f}"], (target, bid, f)
            for f in ACCS:
                assert systems.digest(getattr(sim.accumulators[bid], f)) == want[f"{bid}/{f}"], (target, bid, f)
    acc = np.load(os.path.join(GOLDEN, "kochi6h_acc.npz"))
    for key in acc.files:
        bid, f = key.split("/")
        assert np.array_equal(getattr(sim.accumulators[int(bid)], f), acc[key]), key
    fail = g["failure"]
    assert fail is not None and done == fail["after"]
    with pytest.raises(product.NumericsError) as ei:
        sim.run(fail["within"], threaded=False)
    assert str(ei.value) == fail["message"]
