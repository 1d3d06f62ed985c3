"""Simulation API over the B200 step (SURVEY §8(b) drop-in boundary).

``Simulation(system, settings, plan).run(n_steps, ...)`` keeps the
reference's run-level contract (runner.py:56-378): same constructor, same
``run`` signature and ``RunReport``, ``.states[block_id]`` /
``.accumulators[block_id]`` views, ``.contexts`` with phase logs, re-entrant
``run`` calls, ``on_step`` hooks (serial mode), ``SimulationAborted`` /
``NumericsError`` on non-finite fields.  Behind it, every step is one CUDA
graph replay of the kernels in csrc/ driven through the C ABI; the host only
polls the device error word between chunks of steps.

Accepts the reference's own system/settings/plan objects or this package's
duck-typed equivalents.
"""

from __future__ import annotations

import ctypes
import struct
import time
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .grid import OPPOSITE, lattice_origin, level_abutments
from .schedule import (KIND_CODE, PHASE_CODES, PHASE_ETA, PHASE_FLUX, PHASE_IG_ETA, PHASE_IG_FLUX,
                       SIDE_CODE, build_halo_schedule, build_offset_tables, domain_edges,
                       halo_apply_order, intergrid_segments)

HALO_WIDTH = 2
ROUTINES = ("mass", "momentum", "restrict", "prolong", "halo-eta", "halo-flux", "output")
PHASE_SEQUENCE = ("mass", "restrict", "halo-eta", "momentum", "prolong", "halo-flux", "output", "swap")
TRACE_RECORD = struct.Struct("<IBHHI")        # exchange.py:35


class NumericsError(RuntimeError):
    """A field update produced a non-finite value (kernels.py:23-24)."""


class SimulationAborted(RuntimeError):
    """A rank failed; the run stopped and outputs are not valid (runner.py:43-44)."""


@dataclass
class RankTiming:
    rank: int
    routines: dict
    total: float


@dataclass
class RunReport:
    steps: int
    n_ranks: int
    ranks: list = field(default_factory=list)

    def routine_seconds(self, routine: str) -> list:
        """Per-rank seconds of one routine (report.py:37-38)."""
        return [r.routines.get(routine, 0.0) for r in self.ranks]

    def routine_totals(self):
        out = {r: 0.0 for r in ROUTINES}
        for rt in self.ranks:
            for k, v in rt.routines.items():
                out[k] += v
        return out


@dataclass(eq=False)
class RankContext:
    rank: int
    block_ids: list = field(default_factory=list)
    timers: dict = field(default_factory=lambda: {r: 0.0 for r in ROUTINES})
    phase_log: list = field(default_factory=list)
    wall: float = 0.0


# ------------------------------------------------------------ host setup

def _replicate_halo(a: np.ndarray, g: int = HALO_WIDTH):
    """Edge replication of a ghosted array, rows then columns (kernels.py:108-112)."""
    a[:g] = a[g]
    a[-g:] = a[-g - 1]
    a[:, :g] = a[:, g:g + 1]
    a[:, -g:] = a[:, -g - 1:-g]


def _strip(ni, nj, side, span, sending, g=HALO_WIDTH):
    """Index tuple of a 2-deep eta-shaped strip (exchange.py:162-182)."""
    lo, hi = span
    if side in ("west", "east"):
        if side == "west":
            xs = slice(g, g + 2) if sending else slice(0, g)
        else:
            xs = slice(g + ni - 2, g + ni) if sending else slice(g + ni, g + ni + 2)
        return xs, slice(g + lo, g + hi)
    if side == "south":
        ys = slice(g, g + 2) if sending else slice(0, g)
    else:
        ys = slice(g + nj - 2, g + nj) if sending else slice(g + nj, g + nj + 2)
    return slice(g + lo, g + hi), ys


def h_profile(block):
    """(axis, 1-D profile) when the block's depth depends on one axis only —
    Block.h a broadcast view (stride 0 along the other axis: the synthetic
    coastal-profile and x- or y-only slope kinds) — else None."""
    h = block.h
    if not isinstance(h, np.ndarray) or h.ndim != 2 or h.dtype != np.float64 or h.shape != (block.ni, block.nj):
        return None
    if h.strides[1] == 0:
        return 0, np.ascontiguousarray(h[:, 0])
    if h.strides[0] == 0:
        return 1, np.ascontiguousarray(h[0, :])
    return None


def host_block_arrays(system, settings, pinned: bool = False, device_bathymetry: bool = False):
    """Per block id: ghosted h_ext, optional n_ext, interior eta0 — the
    reference's BlockState setup (kernels.py:39-62, 97-101), initial
    sampling (runner.py:75-80) and fill_bathymetry_halos (exchange.py:281-300).
    ``pinned``: h_ext and eta0 in page-locked memory (ts_host_alloc).
    ``device_bathymetry``: h_ext is None for blocks with a 1-D depth profile
    (h_profile): the device builds it (ts_block_desc.h_profile,
    ts_upload_profiles) and copies every sibling strip; the host then skips
    the strips of the other blocks too."""
    g = HALO_WIDTH
    out = {}
    device_bathymetry = device_bathymetry and any(h_profile(b) is not None for _, b in system.all_blocks())
    for lvl in system.levels:
        for b in lvl.blocks:
            if device_bathymetry and h_profile(b) is not None:
                h = None
            else:
                h = np.empty((b.ni + 2 * g, b.nj + 2 * g))
                h[g:g + b.ni, g:g + b.nj] = np.asarray(b.h, dtype=float)
                _replicate_halo(h)
            if np.ndim(b.manning_n) == 0:
                nman = None
            else:
                nman = np.empty_like(h)
                nman[g:g + b.ni, g:g + b.nj] = np.asarray(b.manning_n, dtype=float)
                _replicate_halo(nman)
            x = b.origin[0] + (np.arange(b.ni) + 0.5) * lvl.dx
            y = b.origin[1] + (np.arange(b.nj) + 0.5) * lvl.dx
            eta0 = np.ascontiguousarray(np.broadcast_to(
                settings.initial.eta0(x[:, None], y[None, :]), (b.ni, b.nj)), dtype=float)
            out[b.block_id] = (h, nman, eta0)
    if pinned:
        for bid, (h, nman, eta0) in out.items():
            ep = N.pinned_empty(eta0.shape)
            ep[...] = eta0
            hp = None
            if h is not None:
                hp = N.pinned_empty(h.shape)
                hp[...] = h
            out[bid] = (hp, nman, ep)
    if device_bathymetry:
        return out
    for lvl in system.levels:
        starts = {b.block_id: lattice_origin(b, lvl.dx) for b in lvl.blocks}
        dims = {b.block_id: (b.ni, b.nj) for b in lvl.blocks}
        for ab in level_abutments(lvl):
            axis = 1 if ab.side in ("west", "east") else 0
            ss = (ab.span[0] - starts[ab.a_id][axis], ab.span[1] - starts[ab.a_id][axis])
            rs = (ab.span[0] - starts[ab.b_id][axis], ab.span[1] - starts[ab.b_id][axis])
            src, dst = out[ab.a_id], out[ab.b_id]
            si = _strip(*dims[ab.a_id], ab.side, ss, True)
            di = _strip(*dims[ab.b_id], OPPOSITE[ab.side], rs, False)
            dst[0][di] = src[0][si]
            if dst[1] is not None and src[1] is not None:
                dst[1][di] = src[1][si]
    return out


# ------------------------------------------------------------ state views

def build_descriptor(system, settings, owner, halo, tables, domain_edges_by_rank, rank=0, world=1, device=0,
                     tile_rows=0):
    """The ts_desc of a configured system (include/tsunami_b200.h; the body
    of Simulation.__init__, runner.py:59-102): per-block arrays from
    host_block_arrays, the halo entries in the reference's apply order, the
    restriction/prolongation segments and the domain-edge rules.  Accepts the
    reference's own objects (duck-typed).  Returns (desc, keepalive)."""
    ordered = system.all_blocks()
    # bathymetry with a 1-D depth profile is built on the device; the
    # siblings' strips are then copied on the device for every block (from
    # whichever h the sender has), so the host skips them
    profiled = any(h_profile(b) is not None for _, b in ordered)
    arrays = host_block_arrays(system, settings, device_bathymetry=profiled)
    keep = []
    blocks = (N.BlockDesc * len(ordered))()
    for k, (lvl, b) in enumerate(ordered):
        h, nman, eta0 = arrays[b.block_id]
        keep += [h, nman, eta0]
        d = blocks[k]
        d.block_id, d.ni, d.nj, d.owner = b.block_id, b.ni, b.nj, owner[k]
        d.level = system.levels.index(lvl)
        d.dx = lvl.dx
        d.manning = float(b.manning_n) if nman is None else 0.0
        if h is None:
            axis, prof = h_profile(b)
            keep.append(prof)
            d.h_ext = None
            d.h_profile = prof.ctypes.data_as(N.PD)
            d.h_axis = axis
        else:
            d.h_ext = h.ctypes.data_as(N.PD)
        d.nman_ext = nman.ctypes.data_as(N.PD) if nman is not None else None
        d.eta0 = eta0.ctypes.data_as(N.PD)
    idx = {b.block_id: k for k, (_, b) in enumerate(ordered)}
    hal = [(idx[e.block_id], idx[e.peer_id], SIDE_CODE[e.side], *e.send_span, *e.recv_span)
           for e in halo_apply_order(halo)]
    eta_segs, flux_segs = intergrid_segments(tables)
    rseg = [(idx[p], idx[c], SIDE_CODE[sg.side], *sg.child_span, sg.ring_start, sg.parent_line, *sg.parent_span)
            for (p, c, sg) in eta_segs]
    pseg = [(idx[p], idx[c], SIDE_CODE[sg.side], *sg.child_span, sg.child_face_line, sg.parent_face_line,
             *sg.parent_span) for (p, c, sg) in flux_segs]
    edges = [(idx[bid], SIDE_CODE[side], KIND_CODE[kind], iv[0], iv[1])
             for r in sorted(domain_edges_by_rank) for (bid, side, iv, kind) in domain_edges_by_rank[r]]
    desc = N.Desc()
    desc.abi_version = N.ABI_VERSION
    desc.n_blocks = len(ordered)
    desc.blocks = blocks
    desc.dt, desc.gravity = float(settings.dt), float(settings.g)
    desc.wet_threshold = float(settings.wet_threshold)
    for name, rows, cls in (("halo", hal, N.HaloEntryC), ("restrict_segs", rseg, N.EtaSegmentC),
                            ("prolong_segs", pseg, N.FluxSegmentC), ("edges", edges, N.EdgeC)):
        arr = (cls * max(1, len(rows)))(*[cls(*r) for r in rows])
        keep.append(arr)
        setattr(desc, name, arr)
    desc.n_halo, desc.n_restrict, desc.n_prolong, desc.n_edges = len(hal), len(rseg), len(pseg), len(edges)
    desc.rank, desc.n_ranks, desc.device, desc.tile_rows = rank, world, device, tile_rows
    keep.append(blocks)
    return desc, keep


class DeviceBlockState:
    """BlockState-shaped view of one device-resident block (kernels.py:31-105).

    Every property returns a host mirror in the reference layout, downloaded
    on first access after a device update.  Mirrors handed out are uploaded
    back before the next device call, so in-place edits such as
    ``st.m_old[:, :] = 1.0`` behave as on the reference's numpy arrays.
    """

    _DEVICE_FIELDS = ("eta_old", "eta_new", "m_old", "m_new", "n_old", "n_new")

    def __init__(self, sim, index, block, thr):
        self._sim, self._index, self._thr = sim, index, thr
        self.block_id, self.ni, self.nj, self.halo = block.block_id, block.ni, block.nj, HALO_WIDTH
        self._mirror = {}
        self._handed = set()

    def _shape(self, name):
        ni, nj = self.ni, self.nj
        return {"eta": (ni + 4, nj + 4), "m_o": (ni + 5, nj + 4), "n_o": (ni + 4, nj + 5),
                "m_n": (ni + 5, nj + 4), "n_n": (ni + 4, nj + 5), "h_e": (ni + 4, nj + 4)}[name[:3]]

    def _get(self, name, hand=True):
        """``hand``: the caller may edit the mirror in place, so it is pushed
        back before the next device call (False for reads made here)."""
        if name not in self._mirror:
            arr = np.empty(self._shape(name))
            N.check(N.lib().ts_get_field(self._sim._h, self._index, N.FIELDS[name],
                                         arr.ctypes.data, arr.size))
            self._mirror[name] = arr
        if hand:
            self._handed.add(name)
        return self._mirror[name]

    eta_old = property(lambda s: s._get("eta_old"))
    eta_new = property(lambda s: s._get("eta_new"))
    m_old = property(lambda s: s._get("m_old"))
    m_new = property(lambda s: s._get("m_new"))
    n_old = property(lambda s: s._get("n_old"))
    n_new = property(lambda s: s._get("n_new"))
    h_ext = property(lambda s: s._get("h_ext"))

    @property
    def wet(self):
        """The reference's stored wet flags, derived: h_ext + eta >= thr for
        the buffer its last writer used (kernels.py:103-105, 155; exchange.py
        :255-257; coupling.py:315) — eta_new within a step, eta_old after the
        step's swap."""
        eta = self._get("eta_old" if self._sim._wet_role == "old" else "eta_new", hand=False)
        return (self._get("h_ext", hand=False) + eta) >= self._thr

    def interior(self, arr):
        g = self.halo
        return arr[g:g + self.ni, g:g + self.nj]

    def _push(self):
        for name in self._handed:
            arr = np.ascontiguousarray(self._mirror[name], dtype=float)
            N.check(N.lib().ts_set_field(self._sim._h, self._index, N.FIELDS[name],
                                         arr.ctypes.data, arr.size))
        self._handed.clear()

    def _invalidate(self):
        self._mirror.clear()
        self._handed.clear()


class DeviceAccumulators:
    """OutputAccumulators view (kernels.py:309-319): max_eta, max_speed,
    max_inundation, each (ni, nj), downloaded on access."""

    def __init__(self, sim, index, block):
        self._sim, self._index, self.ni, self.nj = sim, index, block.ni, block.nj
        self._mirror = {}

    def _get(self, name):
        if name not in self._mirror:
            arr = np.empty((self.ni, self.nj))
            N.check(N.lib().ts_get_field(self._sim._h, self._index, N.FIELDS[name],
                                         arr.ctypes.data, arr.size))
            self._mirror[name] = arr
        return self._mirror[name]

    max_eta = property(lambda s: s._get("max_eta"))
    max_speed = property(lambda s: s._get("max_speed"))
    max_inundation = property(lambda s: s._get("max_inundation"))

    def _invalidate(self):
        self._mirror.clear()


# ------------------------------------------------------------ simulation

class Simulation:
    """A configured system bound to a decomposition plan, resident on a B200.

    ``plan`` is any object with the reference DecompositionPlan interface
    (``n_blocks``, ``n_ranks``, ``rank_of(index)``); its ranks fix the
    exchange apply order and the per-rank report exactly as in the
    reference.  In a single process all blocks live on ``device``.
    """

    def __init__(self, system, settings, plan=None, *, device: int | None = None, tile_rows: int = 0,
                 distributed: bool | None = None, group=None):
        from . import distributed as D
        ordered = system.all_blocks()
        rank, world, local = D.dist_context(group)
        if distributed is None:
            distributed = world > 1
        if not distributed:
            rank, world = 0, 1
        if plan is None:
            from .balance import equal_cell_plan, packed_plan
            cells = [b.ni * b.nj for _, b in ordered]
            plan = equal_cell_plan(cells, 1) if world == 1 else packed_plan(system, world)
        if plan.n_blocks != len(ordered):
            raise ValueError(f"plan covers {plan.n_blocks} blocks, system has {len(ordered)}")
        # one process per GPU: plan rank r is GPU r; a single process runs
        # every rank's blocks on its one GPU (the plan then fixes only the
        # exchange apply order and the per-rank report, as in the reference)
        self.rank, self.world, self.group = rank, world, group
        self.owner = D.owners_from_plan(system, plan, world) if world > 1 else [0] * len(ordered)
        if device is None:
            device = local if world > 1 else 0
        self.system, self.settings, self.plan = system, settings, plan
        self.rank_of = {b.block_id: plan.rank_of(k) for k, (_, b) in enumerate(ordered)}
        self.n_ranks = plan.n_ranks
        self.index = {b.block_id: k for k, (_, b) in enumerate(ordered)}
        self.dx_of = {b.block_id: lvl.dx for lvl, b in ordered}
        self.device = device
        self.halo = build_halo_schedule(system, self.rank_of)
        self.tables = build_offset_tables(system, self.rank_of)
        self.domain_edges = domain_edges(system, settings, self.rank_of)
        self.contexts = [RankContext(rank=r) for r in range(self.n_ranks)]
        for k, (_, b) in enumerate(ordered):
            self.contexts[plan.rank_of(k)].block_ids.append(b.block_id)
        self._h = None
        self._create(ordered, tile_rows)
        if world > 1:
            D.exchange_peer_handles(self._ipc_export, self._ipc_import, rank, world, group)
        thr = settings.wet_threshold
        mine = [(k, b) for k, (_, b) in enumerate(ordered) if self.owner[k] == rank]
        self.states = {b.block_id: DeviceBlockState(self, k, b, thr) for k, b in mine}
        self.accumulators = {b.block_id: DeviceAccumulators(self, k, b) for k, b in mine}
        self.steps_done = 0
        self._wet_role = "new"

    # -- C ABI descriptor -------------------------------------------------
    def _create(self, ordered, tile_rows):
        desc, keep = build_descriptor(self.system, self.settings, self.owner, self.halo, self.tables,
                                      self.domain_edges, self.rank, self.world, self.device, tile_rows)
        hptr = ctypes.c_void_p()
        N.check(N.lib().ts_create(ctypes.byref(desc), ctypes.byref(hptr)))
        self._h = hptr
        self._descr_counts = dict(halo=desc.n_halo, restrict=desc.n_restrict, prolong=desc.n_prolong,
                                  edges=desc.n_edges)
        del keep

    def _ipc_export(self) -> bytes:
        buf = (ctypes.c_char * 256)()
        N.check(N.lib().ts_ipc_export(self._h, buf, 256))
        return bytes(buf)

    def _ipc_import(self, peer: int, blob: bytes):
        buf = (ctypes.c_char * len(blob)).from_buffer_copy(blob)
        N.check(N.lib().ts_ipc_import(self._h, peer, buf, len(blob)))

    def close(self):
        if self._h is not None:
            N.lib().ts_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- running ----------------------------------------------------------
    def _sync_in(self):
        for st in self.states.values():
            st._push()

    def _invalidate(self):
        for st in self.states.values():
            st._invalidate()
        for acc in self.accumulators.values():
            acc._invalidate()

    def _raise_numerics(self, threaded):
        msg = N.lib().ts_last_error().decode()
        blk = ctypes.c_int32(-1)
        N.lib().ts_error_info(self._h, ctypes.byref(blk), None, None, None)
        exc = NumericsError(msg)
        if threaded and self.n_ranks > 1:
            bid = self.system.all_blocks()[blk.value][1].block_id if blk.value >= 0 else None
            rank = self.rank_of.get(bid, 0)
            raise SimulationAborted(f"rank {rank} failed: {msg}") from exc
        raise exc

    def _device_run(self, n, threaded):
        rc = N.lib().ts_run(self._h, n)
        self._invalidate()
        if n:
            self._wet_role = "old"
        if self.world > 1:
            self._distributed_status(rc, threaded)
            return
        if rc == N.TS_ERR_NUMERICS:
            self._raise_numerics(threaded)
        N.check(rc)

    def _distributed_status(self, rc, threaded):
        """Agree on the first failure over ranks (the reference's serial
        order: lowest block, x before y flux, C order) and raise it on all."""
        from . import distributed as D
        local = None
        if rc == N.TS_ERR_NUMERICS:
            blk, what = ctypes.c_int32(-1), ctypes.c_int32(0)
            i, j = ctypes.c_int64(0), ctypes.c_int64(0)
            N.lib().ts_error_info(self._h, ctypes.byref(blk), ctypes.byref(what), ctypes.byref(i),
                                  ctypes.byref(j))
            local = (blk.value, what.value, i.value, j.value)
        elif rc != N.TS_OK:
            local = (-1, 9, 0, 0, N.lib().ts_last_error().decode())
        first = D.first_error(local, self.group)
        if first is None:
            return
        if first[0] < 0:
            raise N.NativeError(N.TS_ERR_CUDA, first[4])
        bid = self.system.all_blocks()[first[0]][1].block_id
        what = ("water level", "x-flux", "y-flux")[first[1]]
        msg = f"non-finite {what} in block {bid} at local cell ({first[2]}, {first[3]})"
        if threaded and self.n_ranks > 1:
            raise SimulationAborted(f"rank {self.rank_of.get(bid, 0)} failed: {msg}") from NumericsError(msg)
        raise NumericsError(msg)

    def run(self, n_steps: int, threaded: bool = True, timeout: float = 60.0,
            trace_path: str | None = None, record_phases: bool = False, on_step=None) -> RunReport:
        """Advance ``n_steps`` steps (runner.py:193-217).  ``threaded`` and
        ``timeout`` are accepted for compatibility; the device runs every
        rank's blocks in one graph either way.  ``on_step(sim, step)``
        requires ``threaded=False`` and runs one step per device call."""
        if threaded and on_step is not None:
            raise ValueError("on_step hooks require the serial scheduler")
        self._sync_in()
        t0 = time.perf_counter()
        routines = {r: 0.0 for r in ROUTINES}
        if on_step is None:
            self._device_run(n_steps, threaded)
            self._accumulate_timings(routines)
        else:
            for step in range(n_steps):
                self._device_run(1, threaded)
                self._accumulate_timings(routines)
                self.steps_done += 1
                on_step(self, step)
                self._sync_in()
            self.steps_done -= n_steps
        wall = time.perf_counter() - t0
        start = self.steps_done
        self.steps_done += n_steps
        if record_phases:
            for ctx in self.contexts:
                ctx.phase_log.extend(list(PHASE_SEQUENCE) * n_steps)
        if trace_path is not None:
            self._write_trace(trace_path, start, n_steps)
        cells = {r: sum(self.system.all_blocks()[self.index[b]][1].cell_count for b in ctx.block_ids)
                 for r, ctx in enumerate(self.contexts)}
        total_cells = max(1, sum(cells.values()))
        ranks = []
        for r, ctx in enumerate(self.contexts):
            share = cells[r] / total_cells
            rt = {k: v * share for k, v in routines.items()}
            for k, v in rt.items():
                ctx.timers[k] += v
            ctx.wall += wall
            ranks.append(RankTiming(rank=r, routines=rt, total=wall))
        return RunReport(steps=n_steps, n_ranks=self.n_ranks, ranks=ranks)

    def _accumulate_timings(self, routines):
        buf = (ctypes.c_double * 7)()
        tot = ctypes.c_double()
        N.check(N.lib().ts_timings(self._h, buf, ctypes.byref(tot)))
        for k, name in enumerate(ROUTINES):
            routines[name] += buf[k]

    def _write_trace(self, path, start, n_steps):
        """The reference's message trace (exchange.py:325-330, 364-370),
        synthesised from the tables: one record per cross-rank payload."""
        msgs = []
        for (s, r, p), n in self.tables.buffer_len.items():
            if s != r:
                msgs.append((PHASE_CODES[p], s, r, n))
        for (s, r, p), n in self.halo.lengths.items():
            if s != r:
                msgs.append((PHASE_CODES[p], s, r, n))
        records = sorted((start + k, *m) for k in range(n_steps) for m in msgs)
        with open(path, "wb") as f:
            for rec in records:
                f.write(TRACE_RECORD.pack(*rec))

    # -- introspection ------------------------------------------------------
    def phase(self, name: str):
        """Run one phase of the step on the device (phase-level tests)."""
        self._sync_in()
        rc = N.lib().ts_phase(self._h, N.PHASES[name])
        self._invalidate()
        self._wet_role = "old" if name == "swap" else "new"
        if rc == N.TS_ERR_NUMERICS:
            self._raise_numerics(False)
        N.check(rc)

    def device_barrier(self):
        """All ranks meet on the device, on the library stream (collective;
        no-op on one rank): what is enqueued next starts within the barrier's
        latency on every rank."""
        N.check(N.lib().ts_device_barrier(self._h))

    def set_timing(self, on: bool):
        N.check(N.lib().ts_set_timing(self._h, 1 if on else 0))

    def kernel_seconds(self):
        m, k, s = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        N.check(N.lib().ts_kernel_seconds(self._h, ctypes.byref(m), ctypes.byref(k), ctypes.byref(s)))
        return m.value, k.value, s.value

    @property
    def stream_ptr(self) -> int:
        """The cudaStream_t all of this simulation's kernels run on."""
        p = ctypes.c_void_p()
        N.check(N.lib().ts_stream(self._h, ctypes.byref(p)))
        return int(p.value or 0)

    def reset(self):
        """A fresh start on the device (as constructing a new Simulation:
        runner.py:59-102): water levels, fluxes and running maxima of the
        owned blocks zeroed, step count 0.  Follow with
        ``upload_initial_state`` to load the initial level."""
        self._sync_in()
        N.check(N.lib().ts_reset(self._h))
        self._invalidate()
        self.steps_done = 0
        self._wet_role = "new"

    def upload_initial_state(self, arrays=None):
        """Copy the host inputs (ghosted bathymetry, initial level) of the
        owned blocks into the device state again — the host->device leg of an
        end-to-end run (BlockState construction + set_initial_eta,
        kernels.py:39-62, 97-101) — in one batched transfer.  ``arrays`` as
        returned by ``host_block_arrays`` (page-locked with ``pinned=True``).
        Returns the bytes copied."""
        if arrays is None:
            arrays = host_block_arrays(self.system, self.settings)
        self._sync_in()
        items = sorted(self.states.items(), key=lambda kv: kv[1]._index)
        n = len(items)
        idx = (ctypes.c_int32 * max(1, n))(*[st._index for _, st in items])
        # blocks whose h_ext is None (host_block_arrays(device_bathymetry=True))
        # send their 1-D depth profile; the device expands it (§8(f)3)
        blocks = {b.block_id: b for _, b in self.system.all_blocks()}
        prof = [(st._index, h_profile(blocks[bid])) for bid, st in items if arrays[bid][0] is None]
        hs = [None if arrays[bid][0] is None else np.ascontiguousarray(arrays[bid][0], dtype=float)
              for bid, _ in items]
        es = [np.ascontiguousarray(arrays[bid][2], dtype=float) for bid, _ in items]
        nbytes = sum(a.nbytes for a in hs if a is not None) + sum(a.nbytes for a in es)
        if prof:
            if any(p is None for _, p in prof):
                raise ValueError("h_ext missing for a block without a 1-D depth profile")
            pi = (ctypes.c_int32 * len(prof))(*[k for k, _ in prof])
            pv = [p[1] for _, p in prof]
            pp = (ctypes.c_void_p * len(prof))(*[a.ctypes.data for a in pv])
            pa = (ctypes.c_int32 * len(prof))(*[p[0] for _, p in prof])
            N.check(N.lib().ts_upload_profiles(self._h, len(prof), pi, pp, pa))
            nbytes += sum(a.nbytes for a in pv)
            if self.world > 1:              # every rank's profiles expanded before any strip is copied
                import torch.distributed as dist
                dist.barrier(self.group)
        hp = (ctypes.c_void_p * max(1, n))(*[0 if a is None else a.ctypes.data for a in hs])
        ep = (ctypes.c_void_p * max(1, n))(*[a.ctypes.data for a in es])
        N.check(N.lib().ts_upload_inputs(self._h, n, idx, hp, ep))
        self._invalidate()
        return nbytes

    # the run's results (the rasters the reference's run writes, cli.py:160-176)
    RESULT_FIELDS = ("max_eta", "max_speed", "max_inundation")
    OUTPUT_FIELDS = RESULT_FIELDS + ("eta_old",)

    def output_buffers(self, pinned: bool = False, fields=OUTPUT_FIELDS):
        """Host buffers for ``download_outputs``: per owned block id one
        array per field (default max_eta, max_speed, max_inundation,
        eta_old), reference shapes."""
        alloc = N.pinned_empty if pinned else np.empty

        def shape(st, f):
            return (st.ni, st.nj) if f.startswith("max") else st._shape(f)

        return {bid: tuple(alloc(shape(st, f)) for f in fields) for bid, st in self.states.items()}

    def download_outputs(self, out=None, fields=None):
        """Device->host read of the results of the owned blocks (by default
        max_eta, max_speed, max_inundation and the current water level; the
        fields are inferred from the buffers' count) in one batched
        transfer.  Fills ``out`` (from ``output_buffers``) when given.
        Returns (dict, bytes)."""
        if out is None:
            out = self.output_buffers()
        self._sync_in()
        items = [(bid, self.states[bid]) for bid in out]
        if fields is None:
            k = len(next(iter(out.values()))) if out else 0
            fields = self.RESULT_FIELDS if k == len(self.RESULT_FIELDS) else self.OUTPUT_FIELDS
        n, nf = len(items), len(fields)
        idx = (ctypes.c_int32 * max(1, n))(*[st._index for _, st in items])
        fld = (ctypes.c_int32 * nf)(*[N.FIELDS[f] for f in fields])
        bufs = [a for bid, _ in items for a in out[bid]]
        for a in bufs:
            if not (a.flags.c_contiguous and a.dtype == np.float64):
                raise ValueError("output buffers must be C-contiguous float64 (use output_buffers)")
        ptr = (ctypes.c_void_p * max(1, len(bufs)))(*[a.ctypes.data for a in bufs])
        N.check(N.lib().ts_download_fields(self._h, n, idx, nf, fld, ptr))
        return out, sum(a.nbytes for a in bufs)

    @property
    def device_bytes(self) -> int:
        return int(N.lib().ts_device_bytes(self._h))

    @property
    def launches_per_step(self) -> int:
        return int(N.lib().ts_launches_per_step(self._h))


def run_simulation(system, settings, plan, n_steps, *, threaded=True, timeout=60.0,
                   trace_path=None, record_phases=False, on_step=None):
    """Build a Simulation, run it, return (sim, report) (runner.py:368-378)."""
    sim = Simulation(system, settings, plan)
    report = sim.run(n_steps, threaded=threaded, timeout=timeout, trace_path=trace_path,
                     record_phases=record_phases, on_step=on_step)
    return sim, report


def read_trace(path):
    with open(path, "rb") as f:
        data = f.read()
    return [TRACE_RECORD.unpack_from(data, o) for o in range(0, len(data), TRACE_RECORD.size)]
