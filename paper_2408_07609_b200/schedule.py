"""Exchange tables of the hot path.

Host-side builders for the three per-step data movements between blocks:

* sibling halo strips (exchange.HaloEntry / HaloSchedule /
  build_halo_schedule, exchange.py:62-159);
* child->parent ring restriction and parent->child face prolongation
  (coupling.EtaSegment / FluxSegment / InterGridLink / IntergridTables /
  build_offset_tables, coupling.py:36-270), including the reference's
  corner rule (west/east rings skip 3 rows) and its first-parent-in-order
  rule for faces on a parent seam (coupling.py:174-202);
* the coarsest-level edge list (runner.py:89-98).

The tables are value-equal to the reference's (tests/test_tables.py checks
them against tables.json dumped from the reference itself) and are then
flattened into the C ABI's ts_halo_entry / ts_eta_segment /
ts_flux_segment / ts_edge records, in the reference's apply order.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .grid import (REFINEMENT_RATIO as R, GridStructureError, lattice_box,
                   lattice_origin, level_abutments, uncovered_side_intervals)

PHASE_ETA = "eta"
PHASE_FLUX = "flux"
PHASE_IG_ETA = "intergrid-eta"
PHASE_IG_FLUX = "intergrid-flux"
PHASE_CODES = {PHASE_ETA: 0, PHASE_FLUX: 1, PHASE_IG_ETA: 2, PHASE_IG_FLUX: 3}
SIDE_CODE = {"west": 0, "east": 1, "south": 2, "north": 3}
KIND_CODE = {"reflective": 0, "radiation": 1}


# ------------------------------------------------------------- halo strips

@dataclass(frozen=True)
class HaloEntry:
    """One edge strip of a rank-pair payload (exchange.py:62-101)."""

    block_id: int
    peer_id: int
    side: str
    send_span: tuple
    recv_span: tuple
    eta_offset: int
    flux_offset: int

    @property
    def span_cells(self) -> int:
        return self.send_span[1] - self.send_span[0]

    @property
    def eta_length(self) -> int:
        return 2 * self.span_cells

    @property
    def flux_length(self) -> int:
        return 4 * self.span_cells + 2

    def element_offset(self, fast: int, slow: int) -> int:
        return fast + 1 + slow * self.span_cells


@dataclass(eq=False)
class HaloSchedule:
    entries: dict = field(default_factory=dict)      # (s, r) -> [HaloEntry]
    lengths: dict = field(default_factory=dict)      # (s, r, phase) -> int

    def expected_senders(self, rank, phase):
        return sorted(s for (s, r, p) in self.lengths if r == rank and p == phase and s != rank)

    def receivers(self, rank, phase):
        return sorted(r for (s, r, p) in self.lengths if s == rank and p == phase and r != rank)


_HALO_SIDE_RANK = {"west": 0, "east": 1, "south": 2, "north": 3}


def build_halo_schedule(system, rank_of=None) -> HaloSchedule:
    if rank_of is None:
        rank_of = {b.block_id: 0 for _, b in system.all_blocks()}
    pairs: dict = {}
    for lvl in system.levels:
        origin = {b.block_id: lattice_origin(b, lvl.dx) for b in lvl.blocks}
        for ab in level_abutments(lvl):
            axis = 1 if ab.side in ("west", "east") else 0
            s0, r0 = origin[ab.a_id][axis], origin[ab.b_id][axis]
            lo, hi = ab.span
            pairs.setdefault((rank_of[ab.a_id], rank_of[ab.b_id]), []).append(
                (ab.a_id, ab.b_id, ab.side, (lo - s0, hi - s0), (lo - r0, hi - r0)))
    sched = HaloSchedule()
    for key, raw in pairs.items():
        raw.sort(key=lambda t: (t[0], _HALO_SIDE_RANK[t[2]], t[3][0]))
        eoff = foff = 0
        out = []
        for (a, b, side, ss, rs) in raw:
            ent = HaloEntry(a, b, side, ss, rs, eoff, foff)
            out.append(ent)
            eoff += ent.eta_length
            foff += ent.flux_length
        sched.entries[key] = out
        sched.lengths[(key[0], key[1], PHASE_ETA)] = eoff
        sched.lengths[(key[0], key[1], PHASE_FLUX)] = foff
    return sched


# --------------------------------------------------------- intergrid tables

@dataclass(frozen=True)
class EtaSegment:
    side: str
    child_span: tuple
    ring_start: int
    parent_line: int
    parent_span: tuple
    offset: int
    length: int


@dataclass(frozen=True)
class FluxSegment:
    side: str
    child_span: tuple
    child_face_line: int
    parent_face_line: int
    parent_span: tuple
    offset: int
    length: int


@dataclass(eq=False)
class InterGridLink:
    parent_block: int
    child_block: int
    eta_segments: list = field(default_factory=list)
    flux_segments: list = field(default_factory=list)


@dataclass(eq=False)
class IntergridTables:
    links: list = field(default_factory=list)
    pair_links: dict = field(default_factory=dict)
    buffer_len: dict = field(default_factory=dict)

    def link_for(self, parent_block, child_block):
        for ln in self.links:
            if ln.parent_block == parent_block and ln.child_block == child_block:
                return ln
        raise KeyError((parent_block, child_block))


def _cover(parents, horizontal, line, lo, hi, faces):
    """Clip the parent-lattice run [lo, hi) on normal coordinate ``line``
    against the parent blocks, in level order; the first parent whose
    normal range contains ``line`` (closed for face lines, half-open for
    cell lines) takes each piece.  Pieces come back sorted by start."""
    todo = [(lo, hi)]
    got = []
    for blk, (x0, y0, x1, y1) in parents:
        along0, along1, n0, n1 = (x0, x1, y0, y1) if horizontal else (y0, y1, x0, x1)
        if not (n0 <= line <= n1 if faces else n0 <= line < n1):
            continue
        rest = []
        for a, b in todo:
            ca, cb = max(a, along0), min(b, along1)
            if ca >= cb:
                rest.append((a, b))
                continue
            got.append((ca, blk, cb, line - n0))
            if a < ca:
                rest.append((a, ca))
            if cb < b:
                rest.append((cb, b))
        todo = rest
        if not todo:
            break
    if todo:
        raise GridStructureError(f"nesting run {todo} at line {line} is not covered by the parent level")
    got.sort(key=lambda g: g[0])
    return [(blk, ca, cb, nl) for (ca, blk, cb, nl) in got]


_RING = {  # side -> (ring_start(ni, nj), ring line in parent cells(ci0, cj0, ni, nj))
    "south": (lambda ni, nj: 0, lambda ci0, cj0, ni, nj: cj0 // R),
    "north": (lambda ni, nj: nj - R, lambda ci0, cj0, ni, nj: (cj0 + nj) // R - 1),
    "west": (lambda ni, nj: 0, lambda ci0, cj0, ni, nj: ci0 // R),
    "east": (lambda ni, nj: ni - R, lambda ci0, cj0, ni, nj: (ci0 + ni) // R - 1),
}
_FACE = {  # side -> (child face line, parent face line)
    "south": (lambda ni, nj: 0, lambda ci0, cj0, ni, nj: cj0 // R),
    "north": (lambda ni, nj: nj, lambda ci0, cj0, ni, nj: (cj0 + nj) // R),
    "west": (lambda ni, nj: 0, lambda ci0, cj0, ni, nj: ci0 // R),
    "east": (lambda ni, nj: ni, lambda ci0, cj0, ni, nj: (ci0 + ni) // R),
}
_SEG_SIDE_RANK = {"south": 0, "north": 1, "west": 2, "east": 3}


def build_offset_tables(system, rank_of=None) -> IntergridTables:
    """Every parent/child transfer segment and its buffer offset (the
    reference's build_offset_tables contract, coupling.py:211-270)."""
    if rank_of is None:
        rank_of = {b.block_id: 0 for _, b in system.all_blocks()}
    raw: dict = {}
    for k in range(1, len(system.levels)):
        lvl, plvl = system.levels[k], system.levels[k - 1]
        abuts = level_abutments(lvl)
        parents = [(pb, lattice_box(pb, plvl.dx)) for pb in plvl.blocks]
        porigin = {pb.block_id: lattice_origin(pb, plvl.dx) for pb in plvl.blocks}
        for child in lvl.blocks:
            ci0, cj0 = lattice_origin(child, lvl.dx)
            ni, nj = child.ni, child.nj
            for side in ("south", "north", "west", "east"):
                horizontal = side in ("south", "north")
                base = ci0 if horizontal else cj0
                for (a, b) in uncovered_side_intervals(lvl, child, side, abuts):
                    if a % R or b % R:
                        raise GridStructureError(
                            f"nesting interface of block {child.block_id} side {side} "
                            f"spans cells [{a}, {b}), not a multiple of {R}")
                    ra, rb = (a, b) if horizontal else (max(a, R), min(b, nj - R))
                    ring0, line_f = _RING[side]
                    if (base + ra) // R < (base + rb) // R:
                        for pb, lo, hi, pl in _cover(parents, horizontal, line_f(ci0, cj0, ni, nj),
                                                     (base + ra) // R, (base + rb) // R, False):
                            off0 = porigin[pb.block_id][0 if horizontal else 1]
                            raw.setdefault((pb.block_id, child.block_id), ([], []))[0].append(
                                EtaSegment(side, (lo * R - base, hi * R - base), ring0(ni, nj), pl,
                                           (lo - off0, hi - off0), -1, hi - lo))
                    cface, pface = _FACE[side]
                    for pb, lo, hi, pl in _cover(parents, horizontal, pface(ci0, cj0, ni, nj),
                                                 (base + a) // R, (base + b) // R, True):
                        off0 = porigin[pb.block_id][0 if horizontal else 1]
                        raw.setdefault((pb.block_id, child.block_id), ([], []))[1].append(
                            FluxSegment(side, (lo * R - base, hi * R - base), cface(ni, nj), pl,
                                        (lo - off0, hi - off0), -1, hi - lo))
    tables = IntergridTables()
    offsets: dict = {}

    def order(seg):
        return (_SEG_SIDE_RANK[seg.side], seg.child_span[0], seg.parent_span[0])

    for (pid, cid) in sorted(raw):
        etas, fluxes = raw[(pid, cid)]
        link = InterGridLink(pid, cid)
        ekey = (rank_of[cid], rank_of[pid], PHASE_IG_ETA)
        fkey = (rank_of[pid], rank_of[cid], PHASE_IG_FLUX)
        for seg in sorted(etas, key=order):
            off = offsets.get(ekey, 0)
            link.eta_segments.append(EtaSegment(seg.side, seg.child_span, seg.ring_start, seg.parent_line,
                                                seg.parent_span, off, seg.length))
            offsets[ekey] = off + seg.length
        for seg in sorted(fluxes, key=order):
            off = offsets.get(fkey, 0)
            link.flux_segments.append(FluxSegment(seg.side, seg.child_span, seg.child_face_line,
                                                  seg.parent_face_line, seg.parent_span, off, seg.length))
            offsets[fkey] = off + seg.length
        tables.links.append(link)
        if link.eta_segments:
            tables.pair_links.setdefault(ekey, []).append(link)
        if link.flux_segments:
            tables.pair_links.setdefault(fkey, []).append(link)
    tables.buffer_len = dict(offsets)
    return tables


def domain_edges(system, settings, rank_of=None) -> dict:
    """{rank: [(block_id, side, (lo, hi), kind)]}: outer-boundary rules on
    the coarsest level only (runner.py:89-98)."""
    l1 = system.levels[0]
    if rank_of is None:
        rank_of = {b.block_id: 0 for _, b in system.all_blocks()}
    ranks = sorted(set(rank_of.values()) | {0})
    out = {r: [] for r in range(max(ranks) + 1)}
    abuts = level_abutments(l1)
    for b in l1.blocks:
        for side in ("west", "east", "south", "north"):
            kind = getattr(settings.boundary, side)
            if kind not in KIND_CODE:
                raise ValueError(f"unknown boundary kind {kind!r}")
            for iv in uncovered_side_intervals(l1, b, side, abuts):
                out[rank_of[b.block_id]].append((b.block_id, side, iv, kind))
    return out


# ------------------------------------------------------- flattening (C ABI)

def halo_apply_order(sched: HaloSchedule):
    """Entries in the reference's apply order: receiver rank, then sorted
    sender rank, then schedule order (runner.py:178-186, 284-291)."""
    out = []
    for rcv in sorted({r for (_, r) in sched.entries}):
        for snd in sorted(s for (s, r) in sched.entries if r == rcv):
            out.extend(sched.entries[(snd, rcv)])
    return out


def intergrid_segments(tables: IntergridTables):
    """(eta segments, flux segments) with their link's blocks, in apply order."""
    eta, flux = [], []
    keys = sorted(tables.pair_links, key=lambda k: (k[1], k[0]))
    for key in keys:
        for link in tables.pair_links[key]:
            if key[2] == PHASE_IG_ETA:
                eta.extend((link.parent_block, link.child_block, s) for s in link.eta_segments)
            else:
                flux.extend((link.parent_block, link.child_block, s) for s in link.flux_segments)
    return eta, flux
