"""Block -> GPU decomposition.

Plans are consecutive runs of the level-ordered block list, as in the
reference (balance.py:102-144): ``DecompositionPlan`` here is value- and
behaviour-compatible, and ``Simulation`` also accepts the reference's own
plan objects.  On top of the reference's equal-cell split this adds an
exact min-max partition under a linear per-block cost model
(cost = slope * cells + intercept, balance.py:31-46), which at 8 GPUs beats
the reference's hill climb.
"""

from __future__ import annotations

import bisect
from dataclasses import dataclass

import numpy as np


class PlanError(ValueError):
    """A decomposition plan is structurally invalid or infeasible."""


class DegenerateFitError(ValueError):
    """Cost samples span fewer than two distinct cell counts."""


@dataclass(frozen=True)
class CostModel:
    """Per-block runtime model in microseconds."""

    slope: float
    intercept: float
    r_squared: float = float("nan")

    def block_cost(self, cells):
        return self.slope * np.asarray(cells, dtype=float) + self.intercept


# The reference's canned GPU coefficients (balance.py:256).
GPU_REFERENCE_MODEL = CostModel(slope=1.09e-4, intercept=46.2, r_squared=0.942)
# B200 step cost of the flattened-tile kernels: blocks share launches, so the
# per-block intercept is only the tile-quantisation tail.
B200_MODEL = CostModel(slope=1.0 / 60.0e3, intercept=0.5)


def fit_cost_model(samples) -> CostModel:
    """Least-squares line through (cells, microseconds) samples; a negative
    intercept is clamped to zero (balance.py:259-284 contract)."""
    pts = np.array([(float(x), float(y)) for x, y in samples], dtype=float).reshape(-1, 2)
    if len(np.unique(pts[:, 0])) < 2:
        raise DegenerateFitError("need samples at at least two distinct cell counts")
    x, y = pts[:, 0], pts[:, 1]
    A = np.stack([x, np.ones_like(x)], axis=1)
    (slope, icept), *_ = np.linalg.lstsq(A, y, rcond=None)
    resid = y - (slope * x + icept)
    ss_res, ss_tot = float(resid @ resid), float(((y - y.mean()) ** 2).sum())
    r2 = (1.0 if ss_res <= 1e-30 else 0.0) if ss_tot == 0 else 1.0 - ss_res / ss_tot
    return CostModel(float(slope), max(0.0, float(icept)), r2)


@dataclass(frozen=True)
class DecompositionPlan:
    """Consecutive assignment: rank r owns blocks [cut[r], cut[r+1])."""

    cells: tuple
    separators: tuple

    def __post_init__(self):
        n = len(self.cells)
        if n == 0:
            raise PlanError("plan needs at least one block")
        prev = 0
        for s in self.separators:
            if not 0 < s < n:
                raise PlanError(f"separator {s} outside (0, {n})")
            if s <= prev:
                raise PlanError("separators must be strictly increasing")
            prev = s

    @property
    def n_blocks(self) -> int:
        return len(self.cells)

    @property
    def n_ranks(self) -> int:
        return len(self.separators) + 1

    def rank_spans(self):
        cuts = (0, *self.separators, len(self.cells))
        return [(cuts[r], cuts[r + 1]) for r in range(self.n_ranks)]

    def rank_of(self, block_index: int) -> int:
        return bisect.bisect_right(self.separators, block_index)

    def blocks_of(self, rank: int) -> range:
        lo, hi = self.rank_spans()[rank]
        return range(lo, hi)


def rank_costs(plan, model: CostModel) -> np.ndarray:
    cuts = (0, *plan.separators, plan.n_blocks)
    cells = np.asarray(plan.cells, dtype=float)
    return np.array([model.slope * cells[a:b].sum() + model.intercept * (b - a)
                     for a, b in zip(cuts[:-1], cuts[1:])])


def predict_rank_cost(plan, model: CostModel, rank: int) -> float:
    return float(rank_costs(plan, model)[rank])


def equal_cell_plan(cells, n_ranks: int) -> DecompositionPlan:
    """The reference's greedy prefix cuts (balance.py:369-393): the r-th cut
    lands where the running total is closest to r/n of the total (first
    such position), keeping one block per remaining rank."""
    cells = tuple(int(c) for c in cells)
    n = len(cells)
    if n_ranks > n:
        raise PlanError(f"{n_ranks} ranks infeasible for {n} blocks")
    if n_ranks < 1:
        raise PlanError("need at least one rank")
    prefix = np.concatenate([[0], np.cumsum(cells)])
    seps, prev = [], 0
    for r in range(1, n_ranks):
        goal = prefix[-1] * r / n_ranks
        cand = np.arange(prev + 1, n - (n_ranks - r) + 1)
        pos = int(cand[np.argmin(np.abs(prefix[cand] - goal))])
        seps.append(pos)
        prev = pos
    return DecompositionPlan(cells, tuple(seps))


# Measured B200 cost per cell (ps) by block width: tools/fit_costs.py
# (single-level systems of 40 M cells of one width, 40 steps; round-1
# kernels).  The march gives a tile ceil((nj+3)/32) warps, or packs tiles of
# nj + 3 threads into 128-thread CTAs (nj = 36), so widths just past a warp
# multiple cost more per cell; the mass pass is per-cell memory work.
B200_MASS_PS_BY_WIDTH = {24: 15.09, 36: 14.2, 48: 13.56, 60: 13.34, 90: 13.36}
B200_MOMENTUM_PS_BY_WIDTH = {24: 36.42, 36: 32.65, 48: 37.49, 60: 29.18, 90: 29.29}
B200_STEP_PS_BY_WIDTH = {24: 54.63, 36: 49.33, 48: 53.05, 60: 44.1, 90: 44.0}


def _lane_factor(nj: int) -> float:
    """Threads the march allots per N-face column (csrc/api.cu tile groups:
    one tile per warp multiple, or tiles packed into 128-thread CTAs)."""
    L = nj + 3
    if L > 128:
        return 128 * ((nj + 1 + 125) // 126) / (nj + 1)
    lanes = 32 * ((L + 31) // 32)
    if (128 // L) * L / 128 > L / lanes + 0.03:
        lanes = 128 / (128 // L)
    return lanes / (nj + 1)


def b200_step_ps_per_cell(nj: int, table=None) -> float:
    """Per-cell step cost of a block of width nj: the measured table, else
    the march's lane utilisation scaled to the table (2/3 of the step is the
    march, 1/3 is per-cell memory work)."""
    table = B200_STEP_PS_BY_WIDTH if table is None else table
    if nj in table:
        return float(table[nj])
    ref = min(table, key=lambda w: abs(w - 60)) if table else 60
    base = float(table.get(ref, 51.4))
    return base * (2.0 * _lane_factor(nj) / _lane_factor(ref) + 1.0) / 3.0


def b200_phase_weights(system):
    """(mass, momentum) B200 cost of every block (global order), ps/step."""
    mass, mom = [], []
    for _, b in system.all_blocks():
        n = b.ni * b.nj
        mass.append(n * B200_MASS_PS_BY_WIDTH.get(b.nj, 13.7))
        if b.nj in B200_MOMENTUM_PS_BY_WIDTH:
            mom.append(n * B200_MOMENTUM_PS_BY_WIDTH[b.nj])
        else:
            mom.append(n * B200_MOMENTUM_PS_BY_WIDTH[60] * _lane_factor(b.nj) / _lane_factor(60))
    return mass, mom


def _phase_objective(seps, mass, mom):
    cuts = (0, *seps, len(mass))
    pm = [sum(mass[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    pk = [sum(mom[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    # the step runs the phases between rank barriers: the slowest rank of
    # each phase sets the pace (ties broken towards the balanced total)
    return max(pm) + max(pk) + 1e-3 * max(x + y for x, y in zip(pm, pk))


def phase_balanced_plan(system, n_ranks: int) -> DecompositionPlan:
    """Consecutive-block plan minimising max(mass) + max(momentum) over
    ranks (the step's two big phases are separated by rank barriers, so
    balancing their sum is not enough): exhaustive for two ranks, else
    separator-wise descent from the min-max plan of the summed cost."""
    cells = tuple(b.ni * b.nj for _, b in system.all_blocks())
    mass, mom = b200_phase_weights(system)
    n = len(cells)
    if n_ranks == 1:
        return DecompositionPlan(cells, ())
    if n_ranks == 2:
        best = min(range(1, n), key=lambda s: _phase_objective((s,), mass, mom))
        return DecompositionPlan(cells, (best,))
    seps = list(minmax_plan(cells, n_ranks, weights=[a + b for a, b in zip(mass, mom)]).separators)
    cur = _phase_objective(seps, mass, mom)
    improved = True
    while improved:
        improved = False
        for k in range(len(seps)):
            lo = seps[k - 1] + 1 if k else 1
            hi = seps[k + 1] - 1 if k + 1 < len(seps) else n - 1
            for v in range(lo, hi + 1):
                if v == seps[k]:
                    continue
                trial = seps[:k] + [v] + seps[k + 1:]
                j = _phase_objective(trial, mass, mom)
                if j < cur - 1e-9:
                    seps, cur, improved = trial, j, True
    return DecompositionPlan(cells, tuple(seps))


@dataclass(frozen=True)
class AssignmentPlan:
    """Any block -> rank assignment (not only consecutive runs): the same
    interface as DecompositionPlan (``n_blocks``, ``n_ranks``, ``rank_of``,
    ``blocks_of``, ``cells``); ``separators`` is None."""

    cells: tuple
    owners: tuple
    ranks: int

    def __post_init__(self):
        if len(self.owners) != len(self.cells) or not self.cells:
            raise PlanError("one owner per block needed")
        if any(not 0 <= o < self.ranks for o in self.owners):
            raise PlanError("owner outside [0, n_ranks)")
        if len(set(self.owners)) != self.ranks:
            raise PlanError("every rank needs at least one block")

    separators = None

    @property
    def n_blocks(self) -> int:
        return len(self.cells)

    @property
    def n_ranks(self) -> int:
        return self.ranks

    def rank_of(self, block_index: int) -> int:
        return self.owners[block_index]

    def blocks_of(self, rank: int) -> list:
        return [k for k, o in enumerate(self.owners) if o == rank]


def packed_plan(system, n_ranks: int, sweeps: int = 50) -> AssignmentPlan:
    """Blocks packed onto ranks without the consecutive-run restriction:
    longest-processing-time placement by mass + momentum cost, then single
    moves and pairwise swaps that lower max(mass) + max(momentum) over ranks
    (the step's two barrier-separated phases).  Cross-rank exchanges cost
    little here (receive areas over NVLink), block granularity a lot."""
    mass, mom = b200_phase_weights(system)
    n = len(mass)
    cells = tuple(b.ni * b.nj for _, b in system.all_blocks())
    if not 1 <= n_ranks <= n:
        raise PlanError(f"{n_ranks} ranks infeasible for {n} blocks")
    owners = [0] * n
    lm, lk = [0.0] * n_ranks, [0.0] * n_ranks
    for k in sorted(range(n), key=lambda k: -(mass[k] + mom[k])):
        r = min(range(n_ranks), key=lambda r: (lm[r] + lk[r], r))
        owners[k] = r
        lm[r] += mass[k]
        lk[r] += mom[k]

    def objective():
        return max(lm) + max(lk) + 1e-3 * max(a + b for a, b in zip(lm, lk))

    cur = objective()
    for _ in range(sweeps):
        improved = False
        for k in range(n):
            a = owners[k]
            for b in range(n_ranks):
                if b == a or (lm[a] - mass[k] <= 0.0 and sum(1 for o in owners if o == a) == 1):
                    continue
                lm[a] -= mass[k]; lk[a] -= mom[k]; lm[b] += mass[k]; lk[b] += mom[k]
                j = objective()
                if j < cur - 1e-9 and any(o == a for i, o in enumerate(owners) if i != k):
                    owners[k], cur, improved = b, j, True
                    break
                lm[a] += mass[k]; lk[a] += mom[k]; lm[b] -= mass[k]; lk[b] -= mom[k]
            a = owners[k]
            for q in range(k + 1, n):
                b = owners[q]
                if b == a:
                    continue
                dm, dk = mass[q] - mass[k], mom[q] - mom[k]
                lm[a] += dm; lk[a] += dk; lm[b] -= dm; lk[b] -= dk
                j = objective()
                if j < cur - 1e-9:
                    owners[k], owners[q], cur, improved = b, a, j, True
                    a = b
                else:
                    lm[a] -= dm; lk[a] -= dk; lm[b] += dm; lk[b] += dk
        if not improved:
            break
    return AssignmentPlan(cells, tuple(owners), n_ranks)


def b200_block_weights(system, table=None, block_overhead_ps: float = 0.0) -> list:
    """Relative B200 step cost of every block (global order), for
    ``minmax_plan(..., weights=...)``: cells x the per-cell cost of the
    block's width (+ a per-block overhead)."""
    return [b.ni * b.nj * b200_step_ps_per_cell(b.nj, table) + block_overhead_ps
            for _, b in system.all_blocks()]


def minmax_plan(cells, n_ranks: int, model: CostModel = B200_MODEL, weights=None) -> DecompositionPlan:
    """Exact minimum of the maximum per-rank cost over all consecutive
    partitions into exactly ``n_ranks`` non-empty runs (O(n^2 k) DP).  The
    per-block cost is ``model.block_cost(cells)``, or ``weights`` when given
    (e.g. ``b200_block_weights``)."""
    cells = tuple(int(c) for c in cells)
    n = len(cells)
    if not 1 <= n_ranks <= n:
        raise PlanError(f"{n_ranks} ranks infeasible for {n} blocks")
    cost = np.asarray(model.block_cost(cells) if weights is None else weights, dtype=float)
    pre = np.concatenate([[0.0], np.cumsum(cost)])
    INF = float("inf")
    best = np.full((n_ranks + 1, n + 1), INF)
    arg = np.zeros((n_ranks + 1, n + 1), dtype=int)
    best[0, 0] = 0.0
    for k in range(1, n_ranks + 1):
        for e in range(k, n - (n_ranks - k) + 1):
            s = np.arange(k - 1, e)
            vals = np.maximum(best[k - 1, s], pre[e] - pre[s])
            q = int(np.argmin(vals))
            best[k, e], arg[k, e] = vals[q], s[q]
    seps, e = [], n
    for k in range(n_ranks, 1, -1):
        e = int(arg[k, e])
        seps.append(e)
    return DecompositionPlan(cells, tuple(sorted(seps)))


def concat_plans(plans) -> DecompositionPlan:
    """Per-level plans joined with forced cuts at level boundaries
    (balance.py:491-503)."""
    cells, seps, off = [], [], 0
    for p in plans:
        cells.extend(p.cells)
        seps.extend(off + s for s in p.separators)
        off += p.n_blocks
        seps.append(off)
    seps.pop()
    return DecompositionPlan(tuple(cells), tuple(seps))
