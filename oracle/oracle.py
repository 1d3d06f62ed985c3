"""TEST INFRASTRUCTURE — Python driver of the C oracle (oracle/swe_oracle.c).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this module, and only as the checker.
The product (``paper_2408_07609_b200``) never imports it.

What is restated here, with the reference file:line each piece follows
(paths relative to /root/reference/pkg/src/blockswe/):

* per-block state setup: BlockState.__init__ / set_initial_eta /
  _replicate_halo (kernels.py:39-112), initial sampling (runner.py:75-84),
  fill_bathymetry_halos (exchange.py:281-300);
* same-level adjacency: level_abutments / uncovered_side_intervals
  (grid.py:340-392);
* the halo schedule: build_halo_schedule (exchange.py:120-159);
* the intergrid offset tables: _segments_for_child / _split_by_parents /
  build_offset_tables (coupling.py:92-270);
* the outer-boundary edge list (runner.py:89-98);
* the apply order of every exchange for a given block->rank map
  (runner.py:146-186, 268-291).

Tables are flattened into int64 op arrays consumed by the C step loop.  The
oracle accepts the reference's own system/settings/plan objects or the
product's duck-typed equivalents.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
G = 2
R = 3
SIDES = ("west", "east", "south", "north")
SIDE_CODE = {s: k for k, s in enumerate(SIDES)}
KIND_CODE = {"reflective": 0, "radiation": 1}
PHASES = ("mass", "restrict", "halo-eta", "momentum", "prolong", "halo-flux",
          "output", "swap")


class OracleNumericsError(RuntimeError):
    """Mirrors kernels.NumericsError (kernels.py:23-24, 115-120)."""


class OracleKernelFault(RuntimeError):
    """Mirrors kernels.KernelFaultError (kernels.py:27-28, 206-211)."""


class OracleStructureError(ValueError):
    """Mirrors grid.GridStructureError raised by the table builders."""


# ---------------------------------------------------------------- C library

def build_library(force: bool = False) -> str:
    """Compile the oracle with gcc (OpenMP, no FMA contraction)."""
    src = os.path.join(HERE, "swe_oracle.c")
    hdr = os.path.join(HERE, "cbrt_oracle.h")
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(src),
                                                   os.path.getmtime(hdr))):
        return LIB_PATH
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-fast-math", "-std=c11", "-o", LIB_PATH + ".tmp", src, "-lm"]
    subprocess.check_call(cmd)
    os.replace(LIB_PATH + ".tmp", LIB_PATH)
    return LIB_PATH


class _OBlock(ctypes.Structure):
    _fields_ = [("ni", ctypes.c_int64), ("nj", ctypes.c_int64),
                ("eta", ctypes.c_void_p * 2), ("m", ctypes.c_void_p * 2),
                ("n", ctypes.c_void_p * 2), ("wet", ctypes.c_void_p),
                ("h", ctypes.c_void_p), ("nman", ctypes.c_void_p),
                ("nman_s", ctypes.c_double), ("dx", ctypes.c_double),
                ("max_eta", ctypes.c_void_p), ("max_speed", ctypes.c_void_p),
                ("max_inund", ctypes.c_void_p), ("block_id", ctypes.c_int64)]


class _OErr(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int64), ("block", ctypes.c_int64),
                ("i", ctypes.c_int64), ("j", ctypes.c_int64),
                ("value", ctypes.c_double)]


class _OSim(ctypes.Structure):
    _fields_ = [("nblocks", ctypes.c_int64), ("blocks", ctypes.POINTER(_OBlock)),
                ("dt", ctypes.c_double), ("grav", ctypes.c_double),
                ("thr", ctypes.c_double), ("cur", ctypes.c_int64),
                ("n_restrict", ctypes.c_int64), ("restrict_ops", ctypes.c_void_p),
                ("n_prolong", ctypes.c_int64), ("prolong_ops", ctypes.c_void_p),
                ("n_halo", ctypes.c_int64), ("halo_ops", ctypes.c_void_p),
                ("n_edges", ctypes.c_int64), ("edge_ops", ctypes.c_void_p),
                ("buf", ctypes.c_void_p), ("accumulate", ctypes.c_int64)]


_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        _LIB = ctypes.CDLL(build_library())
        _LIB.oracle_run.restype = ctypes.c_int64
        _LIB.oracle_phase.restype = ctypes.c_int64
        _LIB.oracle_mass.restype = ctypes.c_int64
        _LIB.oracle_momentum.restype = ctypes.c_int64
        _LIB.oracle_threads.restype = ctypes.c_int64
        _LIB.oracle_threads.argtypes = [ctypes.c_int64]
        _LIB.oracle_cbrt_array.argtypes = [ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_int64]
    return _LIB


def set_threads(n: int = 0) -> int:
    """Set (n > 0) and return the OpenMP thread count of the oracle."""
    return int(lib().oracle_threads(n))


def cbrt(x) -> np.ndarray:
    """The oracle cube root, elementwise (the cbrt-aligned np.cbrt)."""
    a = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(a)
    lib().oracle_cbrt_array(a.ctypes.data, out.ctypes.data, a.size)
    return out if out.ndim else float(out)


class CbrtAlignedNumpy:
    """Proxy for ``numpy`` whose ``cbrt`` is the oracle cube root.

    Monkeypatching ``blockswe.kernels.np`` with this turns the reference into
    the cbrt-aligned reference used to generate golden fixtures.
    """

    def __getattr__(self, name):
        return getattr(np, name)

    @staticmethod
    def cbrt(x):
        return cbrt(x)


# ------------------------------------------------------- geometry (restated)

def cell_start(block, dx):
    """Block.cell_start (grid.py:55-57)."""
    return (int(round(block.origin[0] / dx)), int(round(block.origin[1] / dx)))


def _rect(block, dx):
    i0, j0 = cell_start(block, dx)
    return (i0, j0, i0 + block.ni, j0 + block.nj)


def level_abutments(level):
    """grid.level_abutments (grid.py:340-361): ordered, each contact twice."""
    out = []
    rects = {b.block_id: _rect(b, level.dx) for b in level.blocks}
    opposite = {"east": "west", "west": "east", "north": "south", "south": "north"}
    for a in level.blocks:
        ax0, ay0, ax1, ay1 = rects[a.block_id]
        for b in level.blocks:
            if b.block_id == a.block_id:
                continue
            bx0, by0, bx1, by1 = rects[b.block_id]
            if ax1 == bx0:
                lo, hi = max(ay0, by0), min(ay1, by1)
                if lo < hi:
                    out.append((a.block_id, b.block_id, "east", (lo, hi)))
            if ay1 == by0:
                lo, hi = max(ax0, bx0), min(ax1, bx1)
                if lo < hi:
                    out.append((a.block_id, b.block_id, "north", (lo, hi)))
    return out + [(b, a, opposite[s], sp) for (a, b, s, sp) in out]


def uncovered_side_intervals(level, block, side, abuts=None):
    """grid.uncovered_side_intervals (grid.py:364-392)."""
    i0, j0 = cell_start(block, level.dx)
    if side in ("west", "east"):
        full, local0 = (j0, j0 + block.nj), j0
    else:
        full, local0 = (i0, i0 + block.ni), i0
    if abuts is None:
        abuts = level_abutments(level)
    covered = [sp for (a, _b, s, sp) in abuts if a == block.block_id and s == side]
    pieces = [full]
    for lo, hi in covered:
        nxt = []
        for (p0, p1) in pieces:
            if hi <= p0 or lo >= p1:
                nxt.append((p0, p1))
                continue
            if p0 < lo:
                nxt.append((p0, lo))
            if hi < p1:
                nxt.append((hi, p1))
        pieces = nxt
    return [(p0 - local0, p1 - local0) for (p0, p1) in pieces]


@dataclass(frozen=True)
class HaloOp:
    sender: int        # block id
    receiver: int
    side: str          # sender's side
    send_span: tuple
    recv_span: tuple


def halo_entries(system, rank_of):
    """build_halo_schedule (exchange.py:120-159): {(s_rank, r_rank): [HaloOp]}."""
    side_order = {"west": 0, "east": 1, "south": 2, "north": 3}
    raw = {}
    for lvl in system.levels:
        starts = {b.block_id: cell_start(b, lvl.dx) for b in lvl.blocks}
        for (a, b, side, span) in level_abutments(lvl):
            s0, r0 = starts[a], starts[b]
            k = 1 if side in ("west", "east") else 0
            raw.setdefault((rank_of[a], rank_of[b]), []).append(HaloOp(
                a, b, side, (span[0] - s0[k], span[1] - s0[k]),
                (span[0] - r0[k], span[1] - r0[k])))
    for ents in raw.values():
        ents.sort(key=lambda e: (e.sender, side_order[e.side], e.send_span[0]))
    return raw


def _split_by_parents(parent_rects, horizontal, line_g, lo_g, hi_g, faces=False):
    """coupling._split_by_parents (coupling.py:165-208)."""
    pieces = []
    remaining = [(lo_g, hi_g)]
    for (pb, pi0, pj0, pi1, pj1) in parent_rects:
        if horizontal:
            run0, run1, n0, n1, local_line = pi0, pi1, pj0, pj1, line_g - pj0
        else:
            run0, run1, n0, n1, local_line = pj0, pj1, pi0, pi1, line_g - pi0
        inside = (n0 <= line_g <= n1) if faces else (n0 <= line_g < n1)
        if not inside:
            continue
        nxt = []
        for (a, b) in remaining:
            ca, cb = max(a, run0), min(b, run1)
            if ca >= cb:
                nxt.append((a, b))
                continue
            pieces.append((pb, ca, cb, local_line))
            if a < ca:
                nxt.append((a, ca))
            if cb < b:
                nxt.append((cb, b))
        remaining = nxt
        if not remaining:
            break
    if remaining:
        raise OracleStructureError(
            f"nesting run {remaining} at line {line_g} is not covered by the "
            "parent level")
    pieces.sort(key=lambda p: p[1])
    return pieces


def intergrid_segments(system):
    """_segments_for_child + build_offset_tables link grouping (coupling.py:92-270).

    Returns ``links``: list of (parent_id, child_id, eta_segs, flux_segs) in
    sorted (parent, child) order, segments sorted as the reference sorts
    them.  eta seg = (side, a, b, ring_start, parent_line, pa, pb);
    flux seg = (side, a, b, child_face_line, parent_face_line, pa, pb).
    """
    links = {}
    for k in range(1, len(system.levels)):
        level, parent_level = system.levels[k], system.levels[k - 1]
        abuts = level_abutments(level)
        parent_rects = []
        for pb in parent_level.blocks:
            pi0, pj0 = cell_start(pb, parent_level.dx)
            parent_rects.append((pb, pi0, pj0, pi0 + pb.ni, pj0 + pb.nj))
        for child in level.blocks:
            ci0, cj0 = cell_start(child, level.dx)
            ni, nj = child.ni, child.nj
            for side in ("south", "north", "west", "east"):
                for (a, b) in uncovered_side_intervals(level, child, side, abuts):
                    if (a % R) or (b % R):
                        raise OracleStructureError(
                            f"nesting interface of block {child.block_id} side "
                            f"{side} spans cells [{a}, {b}), not a multiple of {R}")
                    horizontal = side in ("south", "north")
                    ra, rb = (a, b) if horizontal else (max(a, R), min(b, nj - R))
                    if side == "south":
                        ring_start, line_g = 0, cj0 // R
                    elif side == "north":
                        ring_start, line_g = nj - R, (cj0 + nj) // R - 1
                    elif side == "west":
                        ring_start, line_g = 0, ci0 // R
                    else:
                        ring_start, line_g = ni - R, (ci0 + ni) // R - 1
                    base_g = ci0 if horizontal else cj0
                    pa_g, pb_g = (base_g + ra) // R, (base_g + rb) // R
                    if pa_g < pb_g:
                        for (pblk, lo, hi, pline) in _split_by_parents(
                                parent_rects, horizontal, line_g, pa_g, pb_g):
                            pi0, pj0 = cell_start(pblk, parent_level.dx)
                            off0 = pi0 if horizontal else pj0
                            ln = links.setdefault((pblk.block_id, child.block_id), ([], []))
                            ln[0].append((side, lo * R - base_g, hi * R - base_g,
                                          ring_start, pline, lo - off0, hi - off0))
                    if side == "south":
                        face_c, face_g = 0, cj0 // R
                    elif side == "north":
                        face_c, face_g = nj, (cj0 + nj) // R
                    elif side == "west":
                        face_c, face_g = 0, ci0 // R
                    else:
                        face_c, face_g = ni, (ci0 + ni) // R
                    fa_g, fb_g = (base_g + a) // R, (base_g + b) // R
                    for (pblk, lo, hi, fline) in _split_by_parents(
                            parent_rects, horizontal, face_g, fa_g, fb_g, faces=True):
                        pi0, pj0 = cell_start(pblk, parent_level.dx)
                        off0 = pi0 if horizontal else pj0
                        ln = links.setdefault((pblk.block_id, child.block_id), ([], []))
                        ln[1].append((side, lo * R - base_g, hi * R - base_g,
                                      face_c, fline, lo - off0, hi - off0))
    order = {"south": 0, "north": 1, "west": 2, "east": 3}
    out = []
    for key in sorted(links):
        eta, flux = links[key]
        eta.sort(key=lambda s: (order[s[0]], s[1], s[5]))
        flux.sort(key=lambda s: (order[s[0]], s[1], s[5]))
        out.append((key[0], key[1], eta, flux))
    return out


# ---------------------------------------------------------------- the state

class OracleBlockState:
    """Same arrays and buffer roles as kernels.BlockState (kernels.py:31-105)."""

    def __init__(self, block, dx):
        ni, nj = block.ni, block.nj
        self.block_id, self.ni, self.nj, self.halo, self.dx = block.block_id, ni, nj, G, dx
        shape_c = (ni + 4, nj + 4)
        self._eta = [np.zeros(shape_c), np.zeros(shape_c)]
        self._m = [np.zeros((ni + 5, nj + 4)) for _ in range(2)]
        self._n = [np.zeros((ni + 4, nj + 5)) for _ in range(2)]
        self.wet = np.zeros(shape_c, dtype=np.uint8)
        self._cur = 0
        self.h_ext = np.empty(shape_c)
        self.h_ext[G:G + ni, G:G + nj] = np.asarray(block.h, dtype=float)
        _replicate_halo(self.h_ext)
        if np.ndim(block.manning_n) == 0:
            self.n_ext = float(block.manning_n)
        else:
            self.n_ext = np.empty(shape_c)
            self.n_ext[G:G + ni, G:G + nj] = np.asarray(block.manning_n, dtype=float)
            _replicate_halo(self.n_ext)
        self.max_eta = np.zeros((ni, nj))
        self.max_speed = np.zeros((ni, nj))
        self.max_inundation = np.zeros((ni, nj))

    eta_old = property(lambda s: s._eta[s._cur])
    eta_new = property(lambda s: s._eta[1 - s._cur])
    m_old = property(lambda s: s._m[s._cur])
    m_new = property(lambda s: s._m[1 - s._cur])
    n_old = property(lambda s: s._n[s._cur])
    n_new = property(lambda s: s._n[1 - s._cur])

    def interior(self, arr):
        return arr[G:G + self.ni, G:G + self.nj]

    def set_initial_eta(self, eta0, thr):
        self.interior(self._eta[0])[...] = eta0
        self.interior(self._eta[1])[...] = eta0
        self.refresh_wet(thr)

    def refresh_wet(self, thr):
        self.wet[...] = (self.h_ext + self.eta_new) >= thr

    def c_struct(self):
        s = _OBlock()
        s.ni, s.nj = self.ni, self.nj
        for k in range(2):
            s.eta[k] = self._eta[k].ctypes.data
            s.m[k] = self._m[k].ctypes.data
            s.n[k] = self._n[k].ctypes.data
        s.wet = self.wet.ctypes.data
        s.h = self.h_ext.ctypes.data
        if isinstance(self.n_ext, float):
            s.nman, s.nman_s = None, self.n_ext
        else:
            s.nman, s.nman_s = self.n_ext.ctypes.data, 0.0
        s.dx = self.dx
        s.max_eta = self.max_eta.ctypes.data
        s.max_speed = self.max_speed.ctypes.data
        s.max_inund = self.max_inundation.ctypes.data
        s.block_id = self.block_id
        return s


def _replicate_halo(arr):
    """kernels._replicate_halo (kernels.py:108-112)."""
    arr[:G, :] = arr[G:G + 1, :]
    arr[-G:, :] = arr[-G - 1:-G, :]
    arr[:, :G] = arr[:, G:G + 1]
    arr[:, -G:] = arr[:, -G - 1:-G]


# ------------------------------------------------------------ the simulator

class OracleSimulation:
    """CPU oracle of Simulation (runner.py:56-217) with the serial schedule.

    ``rank_of`` (block id -> rank) only changes the apply order of the
    exchanges, exactly as the reference's plan does.  ``eta0`` optionally
    overrides the sampled initial water level per block id (golden fixtures
    carry the reference's own eta0 so np.exp differences between hosts do not
    matter).
    """

    def __init__(self, system, settings, plan=None, rank_of=None, eta0=None,
                 accumulate=True):
        ordered = [(lvl, b) for lvl in system.levels for b in lvl.blocks]
        if plan is not None:
            if plan.n_blocks != len(ordered):
                raise ValueError(f"plan covers {plan.n_blocks} blocks, system has "
                                 f"{len(ordered)}")
            rank_of = {b.block_id: plan.rank_of(k) for k, (_, b) in enumerate(ordered)}
        if rank_of is None:
            rank_of = {b.block_id: 0 for _, b in ordered}
        self.system, self.settings, self.rank_of = system, settings, rank_of
        self.index = {b.block_id: k for k, (_, b) in enumerate(ordered)}
        thr = settings.wet_threshold
        self.states = {}
        for lvl, b in ordered:
            st = OracleBlockState(b, lvl.dx)
            if eta0 is not None and b.block_id in eta0:
                e0 = np.asarray(eta0[b.block_id], dtype=float)
            else:
                x = b.origin[0] + (np.arange(b.ni) + 0.5) * lvl.dx
                y = b.origin[1] + (np.arange(b.nj) + 0.5) * lvl.dx
                e0 = settings.initial.eta0(x[:, None], y[None, :])
            st.set_initial_eta(e0, thr)
            self.states[b.block_id] = st
        self._fill_bathymetry_halos()
        self._build_ops()
        self.blocks = (_OBlock * len(ordered))(
            *[self.states[b.block_id].c_struct() for _, b in ordered])
        self.sim = _OSim()
        self.sim.nblocks = len(ordered)
        self.sim.blocks = self.blocks
        self.sim.dt, self.sim.grav, self.sim.thr = settings.dt, settings.g, thr
        self.sim.cur = 0
        for name in ("restrict", "prolong", "halo", "edge"):
            arr = getattr(self, f"{name}_ops")
            setattr(self.sim, f"n_{name}" if name != "edge" else "n_edges", arr.shape[0])
            setattr(self.sim, f"{name}_ops", arr.ctypes.data if arr.size else None)
        self.buf = np.zeros(max(1, self.buf_len))
        self.sim.buf = self.buf.ctypes.data
        self.sim.accumulate = 1 if accumulate else 0
        self.steps_done = 0

    # exchange.fill_bathymetry_halos (exchange.py:281-300)
    def _fill_bathymetry_halos(self):
        for lvl in self.system.levels:
            starts = {b.block_id: cell_start(b, lvl.dx) for b in lvl.blocks}
            for (a, b, side, span) in level_abutments(lvl):
                src, dst = self.states[a], self.states[b]
                k = 1 if side in ("west", "east") else 0
                ss = (span[0] - starts[a][k], span[1] - starts[a][k])
                rs = (span[0] - starts[b][k], span[1] - starts[b][k])
                opp = {"west": "east", "east": "west", "south": "north", "north": "south"}[side]
                sidx = _eta_strip(src, side, ss, True)
                didx = _eta_strip(dst, opp, rs, False)
                dst.h_ext[didx] = src.h_ext[sidx]
                if not isinstance(dst.n_ext, float) and not isinstance(src.n_ext, float):
                    dst.n_ext[didx] = src.n_ext[sidx]

    def _build_ops(self):
        idx = self.index
        rank_of = self.rank_of
        # halo: apply order = receiver rank, sender rank, schedule order
        ents = halo_entries(self.system, rank_of)
        ops, off = [], 0
        for rcv in sorted({r for (_, r) in ents}):
            for snd in sorted(s for (s, r) in ents if r == rcv):
                for e in ents[(snd, rcv)]:
                    span = e.send_span[1] - e.send_span[0]
                    ops.append([idx[e.sender], idx[e.receiver], SIDE_CODE[e.side],
                                e.send_span[0], e.send_span[1], e.recv_span[0],
                                e.recv_span[1], off, off])
                    off += 2 * span + 2 * (span + 1)
        self.halo_ops = np.array(ops, dtype=np.int64).reshape(-1, 9)
        buf_len = off
        # intergrid: links grouped per (sender, receiver) as in pair_links
        links = intergrid_segments(self.system)
        r_ops, p_ops = [], []
        roff = poff = 0
        rgroups, pgroups = {}, {}
        for (pid, cid, eta, flux) in links:
            pr, cr = rank_of[pid], rank_of[cid]
            if eta:
                rgroups.setdefault((cr, pr), []).append((pid, cid, eta))
            if flux:
                pgroups.setdefault((pr, cr), []).append((pid, cid, flux))
        for rcv in sorted({r for (_, r) in rgroups}):
            for snd in sorted(s for (s, r) in rgroups if r == rcv):
                for (pid, cid, eta) in rgroups[(snd, rcv)]:
                    for (side, a, b, ring, pline, pa, pb) in eta:
                        r_ops.append([idx[cid], idx[pid], SIDE_CODE[side], a, b, ring,
                                      pline, pa, pb, roff])
                        roff += pb - pa
        for rcv in sorted({r for (_, r) in pgroups}):
            for snd in sorted(s for (s, r) in pgroups if r == rcv):
                for (pid, cid, flux) in pgroups[(snd, rcv)]:
                    for (side, a, b, cline, pline, pa, pb) in flux:
                        p_ops.append([idx[pid], idx[cid], SIDE_CODE[side], a, b, cline,
                                      pline, pa, pb, poff])
                        poff += pb - pa
        self.restrict_ops = np.array(r_ops, dtype=np.int64).reshape(-1, 10)
        self.prolong_ops = np.array(p_ops, dtype=np.int64).reshape(-1, 10)
        # outer-boundary edges, coarsest level (runner.py:89-98)
        l1 = self.system.levels[0]
        abuts = level_abutments(l1)
        e_ops = []
        for b in l1.blocks:
            for side in SIDES:
                kind = getattr(self.settings.boundary, side)
                if kind not in KIND_CODE:
                    raise ValueError(f"unknown boundary kind {kind!r}")
                for (lo, hi) in uncovered_side_intervals(l1, b, side, abuts):
                    e_ops.append([idx[b.block_id], SIDE_CODE[side], KIND_CODE[kind], lo, hi])
        self.edge_ops = np.array(e_ops, dtype=np.int64).reshape(-1, 5)
        self.buf_len = max(buf_len, roff, poff)

    # -- running -----------------------------------------------------------
    def _raise(self, rc, err):
        bid = self.system_block_ids()[err.block]
        if rc in (1, 2, 3):
            what = {1: "water level", 2: "x-flux", 3: "y-flux"}[rc]
            raise OracleNumericsError(
                f"non-finite {what} in block {bid} at local cell ({err.i}, {err.j})")
        raise OracleKernelFault(
            f"block {bid}: active face ({err.i}, {err.j}) has non-positive depth "
            f"{err.value:.3e}")

    def system_block_ids(self):
        return [b.block_id for lvl in self.system.levels for b in lvl.blocks]

    def _sync_cur(self):
        for st in self.states.values():
            st._cur = int(self.sim.cur)

    def run(self, n_steps):
        err = _OErr()
        rc = lib().oracle_run(ctypes.byref(self.sim), ctypes.c_int64(n_steps),
                              ctypes.byref(err))
        self._sync_cur()
        if rc:
            self._raise(rc, err)
        self.steps_done += n_steps

    def phase(self, name):
        err = _OErr()
        rc = lib().oracle_phase(ctypes.byref(self.sim), ctypes.c_int64(PHASES.index(name)),
                                ctypes.byref(err))
        self._sync_cur()
        if rc:
            self._raise(rc, err)

    @property
    def accumulators(self):
        return self.states

    def snapshot(self):
        """Every array the reference exposes, per block id (copies)."""
        out = {}
        for bid, st in self.states.items():
            out[bid] = dict(eta_old=st.eta_old.copy(), eta_new=st.eta_new.copy(),
                            m_old=st.m_old.copy(), m_new=st.m_new.copy(),
                            n_old=st.n_old.copy(), n_new=st.n_new.copy(),
                            wet=st.wet.astype(bool), h_ext=st.h_ext.copy(),
                            max_eta=st.max_eta.copy(), max_speed=st.max_speed.copy(),
                            max_inundation=st.max_inundation.copy())
        return out


def _eta_strip(state, side, span, sending):
    """exchange._strip_slices (exchange.py:162-182) as an index tuple."""
    ni, nj = state.ni, state.nj
    lo, hi = span
    if side in ("west", "east"):
        rows = slice(G + lo, G + hi)
        if side == "west":
            cols = slice(G, G + 2) if sending else slice(G - 2, G)
        else:
            cols = slice(G + ni - 2, G + ni) if sending else slice(G + ni, G + ni + 2)
        return (cols, rows)
    cols = slice(G + lo, G + hi)
    if side == "south":
        rows = slice(G, G + 2) if sending else slice(G - 2, G)
    else:
        rows = slice(G + nj - 2, G + nj) if sending else slice(G + nj, G + nj + 2)
    return (cols, rows)


# -------------------------------------------------- single-block kernel calls

def single_block_sim(block, dx, settings, eta0=None):
    """A one-block oracle with no exchanges and no edges, for kernel tests."""
    from types import SimpleNamespace
    lvl = SimpleNamespace(dx=dx, blocks=[block], level_index=1)
    sys_ = SimpleNamespace(levels=[lvl])
    st = SimpleNamespace(dt=settings.dt, g=settings.g,
                         wet_threshold=settings.wet_threshold,
                         boundary=SimpleNamespace(west="reflective", east="reflective",
                                                  south="reflective", north="reflective"),
                         initial=settings.initial)
    sim = OracleSimulation(sys_, st, eta0={block.block_id: eta0} if eta0 is not None else None)
    sim.edge_ops = np.zeros((0, 5), dtype=np.int64)
    sim.sim.n_edges = 0
    return sim
