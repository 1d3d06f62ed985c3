"""Grid-system inputs of the hot path.

Duck-type compatible with the reference's setup types
(/root/reference/pkg/src/blockswe/grid.py:36-158): same class names, field
names and constructor signatures, so systems built with either package run
on either.  Also the same-level adjacency rules the exchange tables are
derived from (grid.py:326-392) and the synthetic Kochi-shaped 5-level
benchmark domain (grid.py:399-525).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

REFINEMENT_RATIO = 3
DEFAULT_GRAVITY = 9.81
DEFAULT_WET_THRESHOLD = 1e-5
DEFAULT_MANNING_N = 0.025
SIDES = ("west", "east", "south", "north")
OPPOSITE = {"west": "east", "east": "west", "south": "north", "north": "south"}


class GridStructureError(ValueError):
    """The system cannot be decomposed into exchange tables (grid.py:28-29)."""


class ScaleUnderflowError(GridStructureError):
    """A scaled Kochi-shaped system would have a block below 3x3 cells."""


@dataclass(eq=False)
class Block:
    """A rectangle of ``ni x nj`` cells; ``h`` is depth (>0 water, <0 land).

    Axis 0 is x, axis 1 is y; ``manning_n`` is a scalar or an (ni, nj)
    array (grid.py:36-60).
    """

    block_id: int
    origin: tuple
    ni: int
    nj: int
    h: np.ndarray
    manning_n: float | np.ndarray = DEFAULT_MANNING_N

    @property
    def cell_count(self) -> int:
        return self.ni * self.nj

    def cell_start(self, dx: float) -> tuple[int, int]:
        return lattice_origin(self, dx)

    def extent(self):
        return (self.origin[0], self.origin[1])


@dataclass(eq=False)
class GridLevel:
    level_index: int
    dx: float
    blocks: list = field(default_factory=list)

    @property
    def cell_count(self) -> int:
        return sum(b.ni * b.nj for b in self.blocks)


@dataclass(eq=False)
class NestedGridSystem:
    """Levels coarsest first; global block order is level-major (grid.py:82-84)."""

    levels: list = field(default_factory=list)

    def all_blocks(self):
        return [(lvl, b) for lvl in self.levels for b in lvl.blocks]

    @property
    def n_blocks(self) -> int:
        return sum(len(lvl.blocks) for lvl in self.levels)

    @property
    def cell_count(self) -> int:
        return sum(lvl.cell_count for lvl in self.levels)

    def level_of_block(self, block_id: int):
        for lvl in self.levels:
            if any(b.block_id == block_id for b in lvl.blocks):
                return lvl
        raise KeyError(f"no block with id {block_id}")


@dataclass(eq=False)
class BoundaryConditions:
    """Coarsest-level edge rule per side: reflective or radiation."""

    west: str = "reflective"
    east: str = "reflective"
    south: str = "reflective"
    north: str = "reflective"

    def __post_init__(self):
        for s in SIDES:
            if getattr(self, s) not in ("reflective", "radiation"):
                raise ValueError(f"unknown boundary kind {getattr(self, s)!r} for {s}")


@dataclass(eq=False)
class InitialCondition:
    """eta0 = A exp(-r^2 / sigma^2) at cell centres, or rest (grid.py:122-141)."""

    kind: str = "rest"
    amplitude: float = 0.0
    sigma: float = 1.0
    center: tuple = (0.0, 0.0)

    def eta0(self, x, y):
        if self.kind == "rest":
            return np.zeros(np.broadcast(x, y).shape)
        if self.kind == "gaussian":
            dist2 = (x - self.center[0]) ** 2 + (y - self.center[1]) ** 2
            return self.amplitude * np.exp(-dist2 / self.sigma ** 2)
        raise ValueError(f"unknown initial condition kind {self.kind!r}")


@dataclass(eq=False)
class SimulationConfig:
    dt: float
    total_duration: float = 0.0
    g: float = DEFAULT_GRAVITY
    wet_threshold: float = DEFAULT_WET_THRESHOLD
    boundary: BoundaryConditions = field(default_factory=BoundaryConditions)
    initial: InitialCondition = field(default_factory=InitialCondition)
    rank_budgets: list | None = None

    @property
    def n_steps(self) -> int:
        return int(round(self.total_duration / self.dt))


# ------------------------------------------------------------------ lattice

def lattice_origin(block, dx: float) -> tuple[int, int]:
    """Block origin in cells of its own level (grid.py:55-57)."""
    return (int(round(block.origin[0] / dx)), int(round(block.origin[1] / dx)))


def lattice_box(block, dx):
    x0, y0 = lattice_origin(block, dx)
    return x0, y0, x0 + block.ni, y0 + block.nj


def cell_centers(block, dx):
    """Cell-centre coordinates (runner.py:77-78)."""
    x = block.origin[0] + (np.arange(block.ni) + 0.5) * dx
    y = block.origin[1] + (np.arange(block.nj) + 0.5) * dx
    return x, y


@dataclass(frozen=True)
class Abutment:
    """Block ``b_id`` touches side ``side`` of ``a_id`` over lattice ``span``."""

    a_id: int
    b_id: int
    side: str
    span: tuple


def level_abutments(level) -> list:
    """Every ordered contact pair of a level (grid.py:340-361 semantics).

    East and north contacts are found first in block order (a outer, b
    inner); the mirrored west/south contacts follow in the same order.
    """
    boxes = [(b.block_id, lattice_box(b, level.dx)) for b in level.blocks]
    forward = []
    for aid, (ax0, ay0, ax1, ay1) in boxes:
        for bid, (bx0, by0, bx1, by1) in boxes:
            if aid == bid:
                continue
            if ax1 == bx0 and max(ay0, by0) < min(ay1, by1):
                forward.append(Abutment(aid, bid, "east", (max(ay0, by0), min(ay1, by1))))
            if ay1 == by0 and max(ax0, bx0) < min(ax1, bx1):
                forward.append(Abutment(aid, bid, "north", (max(ax0, bx0), min(ax1, bx1))))
    mirrored = [Abutment(c.b_id, c.a_id, OPPOSITE[c.side], c.span) for c in forward]
    return forward + mirrored


def _subtract_intervals(full, cuts):
    pieces = [full]
    for lo, hi in cuts:
        nxt = []
        for p0, p1 in pieces:
            if hi <= p0 or lo >= p1:
                nxt.append((p0, p1))
                continue
            if p0 < lo:
                nxt.append((p0, lo))
            if hi < p1:
                nxt.append((hi, p1))
        pieces = nxt
    return pieces


def uncovered_side_intervals(level, block, side, abutments=None) -> list:
    """Local cell intervals of a block side not shared with a sibling
    (grid.py:364-392): physical edges on level 1, nest interfaces below."""
    x0, y0 = lattice_origin(block, level.dx)
    along0, along1 = ((y0, y0 + block.nj) if side in ("west", "east")
                      else (x0, x0 + block.ni))
    abuts = level_abutments(level) if abutments is None else abutments
    shared = [c.span for c in abuts if c.a_id == block.block_id and c.side == side]
    return [(p0 - along0, p1 - along0) for p0, p1 in _subtract_intervals((along0, along1), shared)]


def max_water_depth(level) -> float:
    return max([0.0] + [float(np.max(b.h)) for b in level.blocks if np.size(b.h)])


def cfl_limit(dx: float, dt: float, g: float = DEFAULT_GRAVITY) -> float:
    """Largest depth with dx/dt >= sqrt(2 g h) (grid.py:237-239)."""
    return (dx / dt) ** 2 / (2.0 * g)


def check_system(system, settings) -> list[str]:
    """Structural pre-check of what the device path relies on: positive dt,
    3:1 ratio, lattice alignment, block shapes and the CFL bound (a subset
    of grid.validate_system, grid.py:242-318), in the reference's message
    format (Violation.__str__, grid.py:163-177)."""
    out = []
    if not settings.dt > 0:
        return [f"[timestep] level 0: dt must be positive, got {settings.dt}"]
    for k, lvl in enumerate(system.levels):
        if k and abs(system.levels[k - 1].dx / lvl.dx - REFINEMENT_RATIO) > 1e-9:
            out.append(f"[ratio] level {lvl.level_index}: dx {lvl.dx} is not parent dx "
                       f"{system.levels[k - 1].dx} / {REFINEMENT_RATIO}")
        for b in lvl.blocks:
            if b.ni < 1 or b.nj < 1:
                out.append(f"[shape] level {lvl.level_index} block {b.block_id}: block is {b.ni}x{b.nj}, "
                           "need at least 1x1")
            if np.shape(b.h) != (b.ni, b.nj):
                out.append(f"[bathymetry] level {lvl.level_index} block {b.block_id}: bathymetry shape "
                           f"{np.shape(b.h)} != ({b.ni}, {b.nj})")
        hmax = max_water_depth(lvl)
        if hmax > 0:
            wave = math.sqrt(2.0 * settings.g * hmax)
            if lvl.dx / settings.dt < wave:
                out.append(f"[cfl] level {lvl.level_index}: dx/dt = {lvl.dx / settings.dt:.6g} < "
                           f"sqrt(2 g hmax) = {wave:.6g}")
    return out


def validate_system(system, settings):
    """Light validation report object with ``ok`` and ``violations``."""
    msgs = check_system(system, settings)

    class _Report:
        violations = msgs
        ok = not msgs

        def __str__(self):
            return "all checks passed" if not msgs else "\n".join(msgs)

    return _Report()


# ------------------------------------------- Kochi-shaped 5-level benchmark

# per level: (dx [m], blocks, cells) of the paper's Kochi model (PAPER.md
# Table I, grid.py:400-406), strip heights/widths that factor it at scale 1
KOCHI_LEVELS = ((810.0, 1, 2_012_940), (270.0, 3, 1_703_484), (90.0, 9, 2_230_056),
                (30.0, 11, 9_863_424), (10.0, 60, 31_401_540))
KOCHI_HEIGHTS = (90, 36, 24, 48, 60)
KOCHI_WIDTHS = (22366, 47319, 92919, 205488, 523359)
KOCHI_DEPTH = (4.0, 4000.0)


def _to_multiple(v: float, unit: int) -> int:
    return unit * int(round(v / unit))


def _skewed_split(total: int, n: int, unit: int) -> list[int]:
    """Widths proportional to (k+1)^2, multiples of ``unit``, summing to total."""
    if n == 1:
        return [total]
    wsum = sum((k + 1) ** 2 for k in range(n))
    parts = [max(unit, _to_multiple(total * (k + 1) ** 2 / wsum, unit)) for k in range(n)]
    parts[-1] += total - sum(parts)
    return parts


def kochi_block_inventory(scale: float):
    """[(dx, nj, [(ni, nj), ...]), ...] per level (grid.py:433-470 rules)."""
    if scale <= 0:
        raise ScaleUnderflowError("scale must be positive")
    root = math.sqrt(scale)
    levels = []
    prev = None                                   # (nj, width) of the parent level
    for k, (dx, nblk, cells) in enumerate(KOCHI_LEVELS):
        unit = 1 if k == 0 else REFINEMENT_RATIO
        target = cells * scale
        nj = max(3, _to_multiple(KOCHI_HEIGHTS[k] * root, unit))
        if prev is not None:
            nj = min(nj, REFINEMENT_RATIO * prev[0])
        width = max(unit * nblk, _to_multiple(target / nj, unit))
        if prev is not None and width > REFINEMENT_RATIO * prev[1]:
            cap = REFINEMENT_RATIO * prev[1]
            nj = _to_multiple(math.ceil(target / cap / unit) * unit, unit)
            nj = min(max(nj, unit), REFINEMENT_RATIO * prev[0])
            width = min(cap, max(unit * nblk, _to_multiple(target / nj, unit)))
        if nj < 3 or width < 3 * nblk:
            raise ScaleUnderflowError(
                f"scale {scale} underflows level {k + 1}: cannot fit {nblk} blocks of 3x3")
        widths = _skewed_split(width, nblk, unit)
        for q, w in enumerate(widths):
            if w < 3:
                raise ScaleUnderflowError(
                    f"scale {scale} underflows level {k + 1} block {q + 1}: width {w} < 3")
        levels.append((dx, nj, [(w, nj) for w in widths]))
        prev = (nj, width)
    return levels


def kochi_depth(y, y_center: float, half_extent: float):
    """Cubic coastal ramp: 4 m on the shelf centre to 4000 m offshore
    (grid.py:473-478)."""
    r = np.minimum(1.0, np.abs(y - y_center) / half_extent)
    return KOCHI_DEPTH[0] + (KOCHI_DEPTH[1] - KOCHI_DEPTH[0]) * r ** 3


def build_kochi_scaled_config(scale: float) -> NestedGridSystem:
    """The 5-level 810/270/90/30/10 m Kochi-shaped domain: per level a
    centred east-west chain of abutting strips (1/3/9/11/60 blocks), each
    nested in the previous level's chain; 47,211,444 cells at scale 1.
    Bathymetry depends on y only and is a read-only broadcast view."""
    inv = kochi_block_inventory(scale)
    system = NestedGridSystem()
    bid = 0
    px0 = py0 = 0.0
    for k, (dx, nj, shapes) in enumerate(inv):
        width = sum(w for w, _ in shapes)
        if k:
            pdx, pnj, pshapes = inv[k - 1]
            pwidth = sum(w for w, _ in pshapes)
            px0 += pdx * ((pwidth - width // REFINEMENT_RATIO) // 2)
            py0 += pdx * ((pnj - nj // REFINEMENT_RATIO) // 2)
        level = GridLevel(level_index=k + 1, dx=dx)
        xcur = px0
        for (w, hgt) in shapes:
            bid += 1
            level.blocks.append(Block(bid, (xcur, py0), w, hgt, np.empty(0)))
            xcur += w * dx
        system.levels.append(level)
    l1dx, l1nj, _ = inv[0]
    half = 0.5 * l1nj * l1dx
    yc = 0.0 + half
    for lvl in system.levels:
        for b in lvl.blocks:
            _, ys = cell_centers(b, lvl.dx)
            b.h = np.broadcast_to(kochi_depth(ys, yc, half), (b.ni, b.nj))
    return system


def kochi_settings(system, duration: float = 21600.0, dt: float = 0.2) -> SimulationConfig:
    """save_kochi_config's run settings (config.py:197-208): dt 0.2 s,
    Gaussian 0.5 m hump, sigma = max(fw, fh)/8, centred on the fine level,
    reflective edges; 6 h = 108,000 steps."""
    fine = system.levels[-1]
    fx, fy = fine.blocks[0].origin
    fw = sum(b.ni for b in fine.blocks) * fine.dx
    fh = fine.blocks[0].nj * fine.dx
    return SimulationConfig(dt=dt, total_duration=duration, initial=InitialCondition(
        kind="gaussian", amplitude=0.5, sigma=max(fw, fh) / 8.0,
        center=(fx + fw / 2.0, fy + fh / 2.0)))
