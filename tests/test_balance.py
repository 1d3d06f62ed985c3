"""Decomposition plans and the B200 cost model (balance.py; reference
balance.py:102-293).  CPU only."""

import itertools

import numpy as np
import pytest

import systems


def _max_cost(cost, seps):
    cuts = (0, *seps, len(cost))
    return max(sum(cost[a:b]) for a, b in zip(cuts[:-1], cuts[1:]))


@pytest.mark.parametrize("seed", range(6))
def test_minmax_plan_is_optimal(product, seed):
    rng = np.random.default_rng(seed)
    cells = [int(x) for x in rng.integers(1, 1000, size=int(rng.integers(4, 9)))]
    for nr in range(1, len(cells) + 1):
        plan = product.minmax_plan(cells, nr, model=product.CostModel(slope=1.0, intercept=0.0))
        assert plan.n_ranks == nr and plan.n_blocks == len(cells)
        best = min(_max_cost(cells, s) for s in itertools.combinations(range(1, len(cells)), nr - 1))
        assert _max_cost(cells, plan.separators) == best


def test_minmax_plan_uses_weights(product):
    cells = [100, 100, 100, 100]
    weights = [1.0, 1.0, 1.0, 9.0]
    assert product.minmax_plan(cells, 2, weights=weights).separators == (3,)
    assert product.minmax_plan(cells, 2, model=product.CostModel(1.0, 0.0)).separators == (2,)


def test_plan_errors(product):
    with pytest.raises(product.PlanError):
        product.minmax_plan([1, 2], 3)
    with pytest.raises(product.PlanError):
        product.equal_cell_plan([1, 2], 3)
    with pytest.raises(product.PlanError):
        product.DecompositionPlan((1, 2, 3), (2, 1))


def test_b200_weights_follow_lane_utilisation(product):
    from paper_2408_07609_b200.balance import B200_STEP_PS_BY_WIDTH, b200_step_ps_per_cell
    for w, ps in B200_STEP_PS_BY_WIDTH.items():
        assert b200_step_ps_per_cell(w) == ps
    # a width just past a warp boundary wastes lanes: dearer per cell than
    # one that fills its warps
    assert b200_step_ps_per_cell(30) > b200_step_ps_per_cell(29)
    assert b200_step_ps_per_cell(36) > b200_step_ps_per_cell(60)
    system, _, _ = systems.kochi(product, 0.001)
    w = product.b200_block_weights(system)
    assert len(w) == system.n_blocks and all(x > 0 for x in w)


def test_kochi_plans_balance(product):
    system, _, _ = systems.kochi(product, 1.0)
    cells = [b.cell_count for _, b in system.all_blocks()]
    w = product.b200_block_weights(system)
    for nr, bound in ((2, 1.02), (4, 1.07), (8, 1.16)):
        plan = product.minmax_plan(cells, nr, weights=w)
        cuts = (0, *plan.separators, len(w))
        loads = [sum(w[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
        assert max(loads) / np.mean(loads) < bound, (nr, plan.separators)


def test_fit_cost_model_clamps_intercept(product):
    m = product.fit_cost_model([(100, 10.0), (200, 30.0), (300, 50.0)])
    assert m.slope == pytest.approx(0.2) and m.intercept == 0.0
    m = product.fit_cost_model([(100, 20.0), (200, 30.0), (300, 40.0)])
    assert m.slope == pytest.approx(0.1) and m.intercept == pytest.approx(10.0)


@pytest.mark.parametrize("nr", (2, 3, 4, 8))
def test_phase_balanced_plan_beats_summed_minmax(product, nr):
    """Balancing mass and momentum separately (two barrier-separated
    phases) is never worse than balancing their sum."""
    from paper_2408_07609_b200.balance import _phase_objective
    system, _, _ = systems.kochi(product, 1.0)
    cells = [b.cell_count for _, b in system.all_blocks()]
    mass, mom = product.b200_phase_weights(system)
    p = product.phase_balanced_plan(system, nr)
    q = product.minmax_plan(cells, nr, weights=[a + b for a, b in zip(mass, mom)])
    assert p.n_ranks == nr
    assert _phase_objective(p.separators, mass, mom) <= _phase_objective(q.separators, mass, mom) + 1e-6


@pytest.mark.parametrize("nr", (2, 4, 8))
def test_packed_plan_valid_and_no_worse(product, nr):
    from paper_2408_07609_b200.balance import _phase_objective
    system, _, _ = systems.kochi(product, 1.0)
    mass, mom = product.b200_phase_weights(system)
    p = product.packed_plan(system, nr)
    assert p.n_ranks == nr and p.n_blocks == system.n_blocks and p.separators is None
    assert sorted(k for r in range(nr) for k in p.blocks_of(r)) == list(range(system.n_blocks))
    lm = [sum(mass[k] for k in p.blocks_of(r)) for r in range(nr)]
    lk = [sum(mom[k] for k in p.blocks_of(r)) for r in range(nr)]
    q = product.phase_balanced_plan(system, nr)
    assert max(lm) + max(lk) <= _phase_objective(q.separators, mass, mom) + 1e-6
    ideal = (sum(mass) + sum(mom)) / nr
    assert max(lm) + max(lk) < 1.02 * ideal


def test_assignment_plan_errors(product):
    with pytest.raises(product.PlanError):
        product.AssignmentPlan((1, 2), (0,), 1)
    with pytest.raises(product.PlanError):
        product.AssignmentPlan((1, 2), (0, 2), 2)
    with pytest.raises(product.PlanError):
        product.AssignmentPlan((1, 2), (0, 0), 2)
