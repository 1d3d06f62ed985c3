"""Generate the golden fixtures from the REFERENCE itself.

Runs only where /root/reference exists (the build container); the outputs
are committed under tests/golden/ so the CPU tests can pin the oracle on any
host.  The reference is imported unmodified from /root/reference/pkg/src
and run through its own public API (Simulation, build_halo_schedule,
build_offset_tables, update_mass, ...).  "cbrt-aligned" fixtures are produced
with ``blockswe.kernels.np`` replaced by a proxy whose ``cbrt`` is the
oracle's cube root; "stock" fixtures keep numpy's own
np.cbrt (SVML on this AVX-512 host) for the tolerance check.

    python tests/golden/make_golden.py            # small fixtures (~10 s)
    python tests/golden/make_golden.py --big      # + cfg1/cfg2/kochi digests (~4 min)
"""

import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, HERE)

import blockswe.grid as T                                   # noqa: E402
import blockswe.kernels as K                                # noqa: E402
from blockswe.balance import equal_cell_plan                # noqa: E402
from blockswe.coupling import build_offset_tables           # noqa: E402
from blockswe.exchange import build_halo_schedule           # noqa: E402
from blockswe.grid import uncovered_side_intervals          # noqa: E402
from blockswe.runner import Simulation                      # noqa: E402

import oracle                                               # noqa: E402
import systems                                              # noqa: E402

STOCK_NP = K.np
ALIGNED_NP = oracle.CbrtAlignedNumpy()

FIELDS = ("eta_old", "eta_new", "m_old", "m_new", "n_old", "n_new")
ACCS = ("max_eta", "max_speed", "max_inundation")


def rank_map(system, n_ranks):
    cells = [b.cell_count for _, b in system.all_blocks()]
    plan = equal_cell_plan(cells, n_ranks)
    return plan, {b.block_id: plan.rank_of(k) for k, (_, b) in enumerate(system.all_blocks())}


def tables_of(system, settings, n_ranks):
    plan, rank_of = rank_map(system, n_ranks)
    halo = build_halo_schedule(system, rank_of)
    tabs = build_offset_tables(system, rank_of)
    out = {"n_ranks": n_ranks, "separators": list(plan.separators),
           "halo": [], "halo_lengths": [], "links": [], "pair_links": [],
           "buffer_len": [], "edges": []}
    for (s, r) in sorted(halo.entries):
        out["halo"].append([s, r, [[e.block_id, e.peer_id, e.side, *e.send_span,
                                    *e.recv_span, e.eta_offset, e.flux_offset]
                                   for e in halo.entries[(s, r)]]])
    out["halo_lengths"] = sorted([s, r, p, n] for (s, r, p), n in halo.lengths.items())
    for ln in tabs.links:
        out["links"].append([ln.parent_block, ln.child_block,
                             [[g.side, *g.child_span, g.ring_start, g.parent_line,
                               *g.parent_span, g.offset, g.length] for g in ln.eta_segments],
                             [[g.side, *g.child_span, g.child_face_line, g.parent_face_line,
                               *g.parent_span, g.offset, g.length] for g in ln.flux_segments]])
    for key in sorted(tabs.pair_links):
        out["pair_links"].append([*key, [[ln.parent_block, ln.child_block]
                                         for ln in tabs.pair_links[key]]])
    out["buffer_len"] = sorted([s, r, p, n] for (s, r, p), n in tabs.buffer_len.items())
    l1 = system.levels[0]
    for b in l1.blocks:
        for side in ("west", "east", "south", "north"):
            for iv in uncovered_side_intervals(l1, b, side):
                out["edges"].append([rank_of[b.block_id], b.block_id, side, iv[0], iv[1],
                                     getattr(settings.boundary, side)])
    return out


def run_ref(system, settings, n_steps, n_ranks, aligned=True):
    K.np = ALIGNED_NP if aligned else STOCK_NP
    try:
        plan, _ = rank_map(system, n_ranks)
        sim = Simulation(system, settings, plan)
        sim.run(n_steps, threaded=n_ranks > 1)
    finally:
        K.np = STOCK_NP
    return sim


def state_arrays(sim):
    out = {}
    for bid, st in sim.states.items():
        for f in FIELDS:
            out[f"{bid}/{f}"] = getattr(st, f).copy()
        out[f"{bid}/wet"] = st.wet.copy()
        for f in ACCS:
            out[f"{bid}/{f}"] = getattr(sim.accumulators[bid], f).copy()
    return out


def kernel_cases():
    """Single-block kernel calls on randomised states (fronts, dried cells,
    land, ghosts), cf. tests/test_kernels.py:395-419."""
    out = {}
    for case, per_cell in (("scalar", False), ("percell", True)):
        rng = np.random.default_rng(7 if per_cell else 3)
        ni, nj = 14, 9
        h = rng.uniform(-1.0, 6.0, (ni, nj))
        h[rng.random((ni, nj)) < 0.15] = 2e-6           # sub-threshold films
        nman = 0.01 + 0.05 * rng.random((ni, nj)) if per_cell else 0.03
        blk = T.Block(1, (0.0, 0.0), ni, nj, h, nman)
        eta0 = np.where(h > 0, rng.normal(0.0, 0.3, (ni, nj)), 0.0)
        eta0[rng.random((ni, nj)) < 0.1] = 0.5          # some flooded land
        m0 = rng.normal(0.0, 0.4, (ni + 5, nj + 4))
        n0 = rng.normal(0.0, 0.4, (ni + 4, nj + 5))
        K.np = ALIGNED_NP
        try:
            st = K.BlockState(blk)
            st.set_initial_eta(eta0, 1e-5)
            st.m_old[...] = m0
            st.n_old[...] = n0
            acc = K.OutputAccumulators(ni, nj)
            pre = dict(h=h, eta0=eta0, m0=m0, n0=n0,
                       nman=np.asarray(nman, dtype=float))
            K.update_mass(st, 10.0, 0.2, 1e-5)
            out[f"{case}/mass_eta_new"] = st.eta_new.copy()
            out[f"{case}/mass_wet"] = st.wet.copy()
            K.update_momentum(st, 10.0, 0.2, 9.81, 1e-5)
            out[f"{case}/mom_m_new"] = st.m_new.copy()
            out[f"{case}/mom_n_new"] = st.n_new.copy()
            edges = [("west", "radiation", (1, 7)), ("east", "reflective", None),
                     ("south", "radiation", None), ("north", "radiation", (2, 11))]
            for side, kind, iv in edges:
                K.apply_edge_flux(st, side, kind, iv)
            out[f"{case}/edge_m_new"] = st.m_new.copy()
            out[f"{case}/edge_n_new"] = st.n_new.copy()
            K.accumulate_outputs(st, acc, 1e-5)
            K.accumulate_outputs(st, acc, 1e-5)
            for f in ACCS:
                out[f"{case}/acc_{f}"] = getattr(acc, f).copy()
        finally:
            K.np = STOCK_NP
        for k, v in pre.items():
            out[f"{case}/in_{k}"] = v
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()
    oracle.build_library()

    # 1. tables
    tables = {}
    for name in systems.SMALL + ("kochi", "cfg2"):
        system, settings, _ = systems.make(T, name)
        for nr in (1, 2, 3):
            if nr <= system.n_blocks:
                tables[f"{name}/{nr}"] = tables_of(system, settings, nr)
    sysk, setk, _ = systems.kochi(T, 1.0)
    for nr in (1, 2, 4, 8):
        tables[f"kochi1/{nr}"] = tables_of(sysk, setk, nr)
    with open(os.path.join(HERE, "tables.json"), "w") as f:
        json.dump(tables, f, separators=(",", ":"))

    # 2. small runs, full arrays
    arrays = {}
    for name in systems.SMALL:
        system, settings, n = systems.make(T, name)
        for bid, e0 in systems.eta0_of(system, settings).items():
            arrays[f"{name}/eta0/{bid}"] = e0
        for nr in (1, 2):
            if nr > system.n_blocks:
                continue
            sim = run_ref(system, settings, n, nr)
            for k, v in state_arrays(sim).items():
                arrays[f"{name}/{nr}/aligned/{k}"] = v
        sim = run_ref(system, settings, n, 1, aligned=False)
        for k, v in state_arrays(sim).items():
            arrays[f"{name}/1/stock/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **arrays)

    # 3. kernel calls
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kernel_cases())

    # 4. error messages
    errs = {}
    sysn = T.NestedGridSystem(levels=[T.GridLevel(1, 10.0, [
        systems.flat_block(T, 1, (0.0, 0.0), 8, 8, 30.0),
        T.Block(2, (80.0, 0.0), 8, 8, np.where(np.eye(8, dtype=bool), np.nan, 30.0))])])
    try:
        run_ref(sysn, T.SimulationConfig(dt=0.2), 3, 1)
    except K.NumericsError as exc:
        errs["nan_bathymetry"] = str(exc)
    # wet_threshold 0 over a dry (h = 0, eta = 0) basin: every cell counts as
    # wet, so the reference takes its all-wet branch (kernels.py, `if all_wet:`)
    # and divides 0/0 -- a NumericsError, not a KernelFaultError.
    sysd = T.NestedGridSystem(levels=[T.GridLevel(1, 10.0, [
        T.Block(1, (0.0, 0.0), 6, 5, np.zeros((6, 5)))])])
    try:
        run_ref(sysd, T.SimulationConfig(dt=0.1, wet_threshold=0.0), 3, 1)
    except K.NumericsError as exc:
        errs["dry_basin_threshold0"] = str(exc)
    with open(os.path.join(HERE, "errors.json"), "w") as f:
        json.dump(errs, f, indent=1)

    # 5. bigger configs: digests only
    if args.big:
        dig = {}
        for name, nr in (("kochi", 4), ("cfg1", 1), ("cfg2", 1)):
            system, settings, n = systems.make(T, name)
            d = {"steps": n, "ranks": nr,
                 "eta0": {str(b): systems.digest(e) for b, e in systems.eta0_of(system, settings).items()},
                 "h": {str(b.block_id): systems.digest(b.h) for _, b in system.all_blocks()}}
            for mode in ("aligned", "stock"):
                sim = run_ref(system, settings, n, nr, aligned=(mode == "aligned"))
                arrs = state_arrays(sim)
                d[mode] = {k: systems.digest(v) for k, v in arrs.items() if not k.endswith("/wet")}
                d[mode + "_arrays_max"] = {k: float(np.max(np.abs(v))) for k, v in arrs.items()
                                           if k.split("/")[1] in ACCS}
                if mode == "stock" and name in ("cfg1", "cfg2"):
                    # interior fields for the secondary tolerance check
                    # (SURVEY §8(c) (ii)); cfg2 in float32 to keep the
                    # fixture small (its noise floor is ~1e-4 m anyway)
                    dt_ = np.float64 if name == "cfg1" else np.float32
                    keep = {}
                    for bid, st in sim.states.items():
                        keep[f"{bid}/eta_old"] = st.interior(st.eta_old).astype(dt_)
                        for f in ("max_eta", "max_inundation"):
                            keep[f"{bid}/{f}"] = getattr(sim.accumulators[bid], f).astype(dt_)
                    np.savez_compressed(os.path.join(HERE, f"{name}_stock.npz"), **keep)
            dig[name] = d
            print(name, "done", flush=True)
        with open(os.path.join(HERE, "digests.json"), "w") as f:
            json.dump(dig, f, indent=1)


if __name__ == "__main__":
    main()
