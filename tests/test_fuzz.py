"""Random nested systems (systems.random_nested): the oracle against the
reference's own digests (tests/golden/fuzz.json, make_golden_fuzz.py), and
the CUDA path against the oracle, bitwise, on the same systems and plans.

Each system mixes what the fixed fixtures cover one at a time: ragged
sibling spans on every level, children touching the parent level's edge,
straddling parent seams and abutting each other, three levels with a child
inside a child, wet/dry fronts, zero / scalar / per-cell Manning, mixed
edge kinds and 1-3 ranks' apply orders.
"""

import json
import os

import numpy as np
import pytest

import systems
from conftest import GOLDEN

with open(os.path.join(GOLDEN, "fuzz.json")) as _f:
    FUZZ = json.load(_f)
SEEDS = sorted(int(k) for k in FUZZ)
ACCS = ("max_eta", "max_speed", "max_inundation")
FIELDS = ("eta_old", "eta_new", "m_old", "m_new", "n_old", "n_new")


def _digests(sim):
    out = {}
    for bid, st in sim.states.items():
        for f in FIELDS:
            out[f"{bid}/{f}"] = systems.digest(getattr(st, f))
    for bid, acc in sim.accumulators.items():
        for f in ACCS:
            out[f"{bid}/{f}"] = systems.digest(getattr(acc, f))
    return out


def _case(product, seed):
    system, settings, n, nr = systems.random_nested(product, seed)
    plan = product.equal_cell_plan([b.cell_count for _, b in system.all_blocks()], nr)
    return system, settings, n, plan, FUZZ[str(seed)]


def _check(sim, run, n, want, NumericsError):
    if want["error"] is not None:
        with pytest.raises(NumericsError) as ei:
            run(n)
        assert str(ei.value) == want["error"]
        return
    run(n)
    got = _digests(sim)
    bad = sorted(k for k, v in want["digests"].items() if got.get(k) != v)
    assert not bad, f"{len(bad)} arrays differ from the reference, first {bad[:4]}"


def test_fuzz_fixture_shape():
    assert len(SEEDS) >= 24
    assert any(len(d["blocks"]) == 3 for d in FUZZ.values())
    assert {d["ranks"] for d in FUZZ.values()} == {1, 2, 3}


@pytest.mark.parametrize("seed", SEEDS)
def test_oracle_vs_reference_fuzz(oracle_mod, product, seed):
    system, settings, n, plan, want = _case(product, seed)
    orc = oracle_mod.OracleSimulation(system, settings, plan)
    _check(orc, orc.run, n, want, product.NumericsError)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS)
def test_gpu_vs_reference_fuzz(cuda_device, oracle_mod, product, seed):
    """Digests against the reference, then every array against the oracle
    (for a readable first difference if the digests disagree)."""
    system, settings, n, plan, want = _case(product, seed)
    gpu = product.Simulation(system, settings, plan)
    try:
        if want["error"] is not None:
            _check(gpu, lambda k: gpu.run(k, threaded=False), n, want, product.NumericsError)
            return
        orc = oracle_mod.OracleSimulation(system, settings, plan)
        for chunk in (1, n // 2 - 1, n - n // 2):
            gpu.run(chunk, threaded=False)
            orc.run(chunk)
        for bid, o in orc.states.items():
            g = gpu.states[bid]
            for f in FIELDS:
                a, b = getattr(g, f), getattr(o, f)
                assert np.array_equal(a, b, equal_nan=True), (seed, bid, f, np.argwhere(a != b)[:3].tolist())
            for f in ACCS:
                assert np.array_equal(getattr(gpu.accumulators[bid], f), getattr(o, f)), (seed, bid, f)
        got = _digests(gpu)
        assert all(got[k] == v for k, v in want["digests"].items())
    finally:
        gpu.close()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", SEEDS[::3])
def test_gpu_vs_oracle_fuzz_packed_plan(cuda_device, oracle_mod, product, seed):
    """The same systems under packed_plan (non-consecutive block -> rank
    map, the bench's multi-GPU plan) for 2 and 3 ranks' apply orders."""
    system, settings, n, _, _ = _case(product, seed)
    for nr in (2, 3):
        if nr > system.n_blocks:
            continue
        plan = product.packed_plan(system, nr)
        gpu = product.Simulation(system, settings, plan)
        orc = oracle_mod.OracleSimulation(system, settings, plan)
        try:
            gpu.run(n, threaded=False)
            orc.run(n)
            assert _digests(gpu) == _digests(orc), (seed, nr)
        finally:
            gpu.close()
