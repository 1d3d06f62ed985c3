"""Deterministic test systems shared by the golden generator and the tests.

``make(T, name)`` builds ``(system, settings, n_steps)`` from a namespace
``T`` exposing the reference's constructor signatures (Block, GridLevel,
NestedGridSystem, SimulationConfig, BoundaryConditions, InitialCondition) —
either ``blockswe.grid`` (golden generation, this container only) or the
product's ``paper_2408_07609_b200.grid`` (tests, any host).  Geometry and
bathymetry use only exact IEEE elementwise arithmetic, so they are
host-independent; eta0 uses np.exp, so the fixtures carry it explicitly.
"""

import numpy as np


def flat_block(T, block_id, origin, ni, nj, depth, manning_n=0.025):
    """tests/conftest.py:15-17"""
    return T.Block(block_id=block_id, origin=origin, ni=ni, nj=nj,
                   h=np.full((ni, nj), float(depth)), manning_n=manning_n)


def hump(T, amplitude, sigma, center, dt=0.2, **kw):
    """tests/conftest.py:64-66"""
    return T.SimulationConfig(dt=dt, initial=T.InitialCondition(
        kind="gaussian", amplitude=amplitude, sigma=sigma, center=center), **kw)


def slope(origin, ni, nj, dx, d0, gx, gy=0.0):
    """config._build_bathymetry 'slope' (config.py:47-53)."""
    x = origin[0] + (np.arange(ni) + 0.5) * dx
    y = origin[1] + (np.arange(nj) + 0.5) * dx
    return d0 + gx * x[:, None] + gy * y[None, :] + np.zeros((ni, nj))


def beach(T):
    """Single 48x40 block, sloping beach with dry land, radiation W/N."""
    x = (np.arange(48) + 0.5) * 10.0
    h = np.broadcast_to((8.0 - 0.02 * x)[:, None], (48, 40)).copy()
    system = T.NestedGridSystem(levels=[T.GridLevel(1, 10.0, [T.Block(1, (0.0, 0.0), 48, 40, h)])])
    settings = T.SimulationConfig(
        dt=0.2, boundary=T.BoundaryConditions(west="radiation", north="radiation"),
        initial=T.InitialCondition("gaussian", 0.6, 60.0, (200.0, 150.0)))
    return system, settings, 300


def two_parent(T):
    """tests/conftest.py:36-47 with a hump."""
    system = T.NestedGridSystem(levels=[
        T.GridLevel(1, 9.0, [flat_block(T, 1, (0.0, 0.0), 6, 6, 8.0),
                             flat_block(T, 2, (54.0, 0.0), 6, 6, 8.0)]),
        T.GridLevel(2, 3.0, [flat_block(T, 3, (18.0, 9.0), 18, 12, 8.0)])])
    return system, hump(T, 0.4, 18.0, (54.0, 27.0)), 50


def identity3(T):
    """Three coincident levels: every block is both parent and child (the
    read-all-then-write hazard)."""
    system = T.NestedGridSystem(levels=[
        T.GridLevel(1, 27.0, [flat_block(T, 1, (0.0, 0.0), 4, 4, 8.0)]),
        T.GridLevel(2, 9.0, [flat_block(T, 2, (0.0, 0.0), 12, 12, 8.0)]),
        T.GridLevel(3, 3.0, [flat_block(T, 3, (0.0, 0.0), 36, 36, 8.0)])])
    return system, hump(T, 0.4, 30.0, (50.0, 60.0)), 60


def quad_wetdry(T):
    """Four sibling blocks with ragged west/east AND south/north spans (so
    tangential strips overlap at span ends), a coastline with dry land,
    per-cell Manning on one block, a nested child straddling all four
    parents across two seams, radiation on west and north."""
    dx = 30.0

    def blk(bid, o, ni, nj, nman=0.025):
        return T.Block(bid, o, ni, nj, slope(o, ni, nj, dx, 10.0, -0.011), nman)

    rng = np.random.default_rng(42)
    n4 = 0.02 + 0.02 * rng.random((18, 9))
    lv1 = T.GridLevel(1, dx, [blk(1, (0.0, 0.0), 24, 12), blk(2, (720.0, 0.0), 15, 12),
                              blk(3, (0.0, 360.0), 21, 9), blk(4, (630.0, 360.0), 18, 9, n4)])
    lv2 = T.GridLevel(2, 10.0, [T.Block(5, (540.0, 240.0), 36, 36,
                                        slope((540.0, 240.0), 36, 36, 10.0, 10.0, -0.011))])
    system = T.NestedGridSystem(levels=[lv1, lv2])
    settings = T.SimulationConfig(
        dt=0.2, boundary=T.BoundaryConditions(west="radiation", north="radiation"),
        initial=T.InitialCondition("gaussian", 0.5, 150.0, (760.0, 330.0)))
    return system, settings, 150


def chain(T):
    """tests/conftest.py:50-56 with a hump (halo workhorse)."""
    system = T.NestedGridSystem(levels=[T.GridLevel(1, 10.0, [
        flat_block(T, 1, (0.0, 0.0), 8, 10, 40.0),
        flat_block(T, 2, (80.0, 0.0), 12, 10, 40.0),
        flat_block(T, 3, (220.0, 0.0), 6, 10, 40.0)])])
    return system, hump(T, 0.5, 260.0 / 6, (130.0, 50.0)), 60


def kochi(T, scale=0.001):
    """build_kochi_scaled_config (grid.py:481-525) with the acceptance-test
    hump (tests/test_acceptance.py:48-57)."""
    system = T.build_kochi_scaled_config(scale)
    fine = system.levels[-1]
    fw = sum(b.ni for b in fine.blocks) * fine.dx
    fh = fine.blocks[0].nj * fine.dx
    settings = hump(T, 0.5, fw / 8, (fine.blocks[0].origin[0] + fw / 2,
                                     fine.blocks[0].origin[1] + fh / 2))
    return system, settings, 30


def cfg1(T):
    """256^2 sloping beach, 1000 steps."""
    h = slope((0.0, 0.0), 256, 256, 10.0, 20.0, -0.01)
    system = T.NestedGridSystem(levels=[T.GridLevel(1, 10.0, [T.Block(1, (0.0, 0.0), 256, 256, h, 0.025)])])
    settings = T.SimulationConfig(dt=0.2, total_duration=200.0, g=9.81, wet_threshold=1e-5,
                                  initial=T.InitialCondition("gaussian", 0.3, 200.0, (1200.0, 1280.0)))
    return system, settings, 1000


def cfg2(T):
    """2-level 270 -> 90 m with wet/dry, 2000 steps."""
    h1 = slope((0.0, 0.0), 240, 240, 270.0, 180.0, -0.005)
    h2 = slope((16200.0, 16200.0), 360, 360, 90.0, 180.0, -0.005)
    system = T.NestedGridSystem(levels=[
        T.GridLevel(1, 270.0, [T.Block(1, (0.0, 0.0), 240, 240, h1, 0.025)]),
        T.GridLevel(2, 90.0, [T.Block(2, (16200.0, 16200.0), 360, 360, h2, 0.025)])])
    settings = T.SimulationConfig(
        dt=0.2, total_duration=400.0,
        boundary=T.BoundaryConditions(west="radiation"),
        initial=T.InitialCondition("gaussian", 2.0, 3000.0, (33000.0, 32400.0)))
    return system, settings, 2000


def cfg5(T, scale=1.0, strips=8, rows=None):
    """one 10 m level of n x n cells (n = 20000 at scale
    1, 400 M cells) as ``strips`` abutting x-strips; 50 m deep except the
    last strip, a slope whose coast sits at 90 % of the x extent; a 0.3 m
    hump near the coast.  ``rows``: rows per strip instead (weak scaling:
    one 2500 x 20000 strip per GPU)."""
    nj = int(round(20000 * scale))
    if rows is None:
        n = nj - nj % strips
        nj, ni = n, n // strips
    else:
        ni = int(rows)
    dx = 10.0
    wx, wy = strips * ni * dx, nj * dx
    x_last = (strips - 1) * ni * dx           # the last strip: 50 m deep at its start, then 1 %
    blocks = []
    for k in range(strips):
        o = (k * ni * dx, 0.0)
        # x-only depths as broadcast views (the same values as full arrays;
        # the product builds such bathymetry on the device, runner.h_profile)
        if k < strips - 1:
            h = np.broadcast_to(np.full((ni, 1), 50.0), (ni, nj))
        else:
            h = np.broadcast_to(slope(o, ni, 1, dx, 50.0 + 0.01 * x_last, -0.01), (ni, nj))
        blocks.append(T.Block(k + 1, o, ni, nj, h, 0.025))
    system = T.NestedGridSystem(levels=[T.GridLevel(1, dx, blocks)])
    sigma = 0.01 * max(wx, wy)
    settings = T.SimulationConfig(
        dt=0.2, total_duration=40.0,
        initial=T.InitialCondition("gaussian", 0.3, sigma, (x_last + 0.5 * sigma, 0.5 * wy)))
    return system, settings, 200


class BumpInitial:
    """Compact bump A * max(0, 1 - r^2/s^2)^2: only IEEE elementwise
    arithmetic, so eta0 is the same on every host (unlike np.exp).  Duck-
    types InitialCondition for runner.py:77-80 (``eta0(x, y)``)."""

    kind = "bump"

    def __init__(self, amplitude, sigma, center):
        self.amplitude, self.sigma, self.center = float(amplitude), float(sigma), center

    def eta0(self, x, y):
        cx, cy = self.center
        r2 = (x - cx) * (x - cx) + (y - cy) * (y - cy)
        q = np.maximum(0.0, 1.0 - r2 / (self.sigma * self.sigma))
        return self.amplitude * (q * q)


def _split(rng, rect, unit, n_max):
    """Guillotine split of a cell rect (x, y, w, h) into at most n_max
    rects whose sides are multiples of ``unit`` (and >= unit)."""
    rects = [rect]
    while len(rects) < n_max and rng.random() < 0.75:
        k = int(rng.integers(len(rects)))
        x, y, w, h = rects[k]
        axis = int(rng.integers(2))
        size = (w, h)[axis]
        if size < 2 * unit:
            continue
        cut = unit * int(rng.integers(1, size // unit))
        if axis == 0:
            rects[k:k + 1] = [(x, y, cut, h), (x + cut, y, w - cut, h)]
        else:
            rects[k:k + 1] = [(x, y, w, cut), (x, y + cut, w, h - cut)]
    return rects


def random_nested(T, seed):
    """A random valid 2- or 3-level nested system (3:1, lattice-aligned,
    enclosed): guillotine-split sibling blocks with ragged spans on every
    level, children anywhere inside the parent level (touching its edge,
    straddling parent seams, abutting each other), sloping bathymetry with
    land and wet/dry fronts, scalar / zero / per-cell Manning, random edge
    kinds, a compact bump.  Returns (system, settings, n_steps, n_ranks)."""
    rng = np.random.default_rng(1000 + seed)
    dx1 = 90.0
    nx, ny = int(rng.integers(9, 31)), int(rng.integers(9, 31))
    # a plane beach: depth 0 on a line through a random point (all wet in
    # a third of the systems), slope 0.3-1.2 %, any direction
    sl, th = rng.uniform(0.003, 0.012), rng.uniform(0.0, 2.0 * np.pi)
    gx, gy = float(-sl * np.cos(th)), float(-sl * np.sin(th))
    px, py = rng.uniform(0.0, nx * dx1), rng.uniform(0.0, ny * dx1)
    d0 = float(-gx * px - gy * py + (rng.uniform(40.0, 60.0) if rng.random() < 0.33 else 0.0))
    manning = (0.0, 0.025, 0.03)
    bid = [0]

    def blocks_of(rects, dx, unit_cells):
        out = []
        for (x, y, w, h) in _split(rng, rects, unit_cells, 3):
            bid[0] += 1
            o = (x * dx, y * dx)
            hb = slope(o, w, h, dx, d0, gx, gy)
            nm = manning[int(rng.integers(3))]
            if rng.random() < 0.25:
                nm = 0.01 + 0.03 * rng.random((w, h))
            out.append(T.Block(bid[0], o, w, h, hb, nm))
        return out

    levels = [T.GridLevel(1, dx1, blocks_of((0, 0, nx, ny), dx1, 3))]
    # level 2: one or two non-overlapping child rects (parent cells)
    kids = []
    for _ in range(int(rng.integers(1, 3))):
        for _try in range(20):
            pw, ph = int(rng.integers(2, max(3, nx // 2))), int(rng.integers(2, max(3, ny // 2)))
            px, py = int(rng.integers(0, nx - pw + 1)), int(rng.integers(0, ny - ph + 1))
            if all(px >= a + c or a >= px + pw or py >= b + d or b >= py + ph for a, b, c, d in kids):
                kids.append((px, py, pw, ph))
                break
    lv2 = []
    for (px, py, pw, ph) in kids:
        lv2 += blocks_of((3 * px, 3 * py, 3 * pw, 3 * ph), dx1 / 3, 3)
    levels.append(T.GridLevel(2, dx1 / 3, lv2))
    if rng.random() < 0.5:
        px, py, pw, ph = kids[0]                       # level-2 cells inside the first child rect
        w, h = int(rng.integers(1, 3 * pw + 1)), int(rng.integers(1, 3 * ph + 1))
        x, y = 3 * px + int(rng.integers(0, 3 * pw - w + 1)), 3 * py + int(rng.integers(0, 3 * ph - h + 1))
        levels.append(T.GridLevel(3, dx1 / 9, blocks_of((3 * x, 3 * y, 3 * w, 3 * h), dx1 / 9, 3)))
    system = T.NestedGridSystem(levels=levels)
    kinds = ("reflective", "radiation")
    bc = T.BoundaryConditions(**{s: kinds[int(rng.integers(2))] for s in ("west", "east", "south", "north")})
    cx, cy = rng.uniform(0.0, nx * dx1), rng.uniform(0.0, ny * dx1)
    settings = T.SimulationConfig(dt=0.2, boundary=bc, initial=BumpInitial(
        rng.uniform(0.3, 1.5), rng.uniform(300.0, 1500.0), (cx, cy)))
    n_ranks = int(rng.integers(1, 4))
    return system, settings, 100, min(n_ranks, system.n_blocks)


SMALL = ("beach", "two_parent", "identity3", "quad_wetdry", "chain")
ALL = SMALL + ("kochi", "cfg1", "cfg2")


def make(T, name):
    return globals()[name](T)


def eta0_of(system, settings):
    """Initial sampling (runner.py:75-80) per block id."""
    out = {}
    for lvl in system.levels:
        for b in lvl.blocks:
            x = b.origin[0] + (np.arange(b.ni) + 0.5) * lvl.dx
            y = b.origin[1] + (np.arange(b.nj) + 0.5) * lvl.dx
            out[b.block_id] = np.asarray(settings.initial.eta0(x[:, None], y[None, :]), dtype=float)
    return out


def digest(arr) -> str:
    """sha256 of a float array with -0.0 canonicalised to +0.0."""
    import hashlib
    a = np.ascontiguousarray(np.asarray(arr, dtype=np.float64) + 0.0)
    return hashlib.sha256(a.tobytes()).hexdigest()[:32]
