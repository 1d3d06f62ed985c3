"""Benchmark: Gcell-updates/s of the nested-grid tsunami step on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config kochi|cfg1|cfg2|cfg5|cfg5weak] [--scale S]

Workload (BASELINE.json ``metric`` / configs[2]): the 5-level 810/270/90/30/10 m
Kochi-shaped domain, 47,211,444 cells, dt 0.2 s (a 6-h simulation is 108,000
steps), synthetic bathymetry and a 0.5 m Gaussian source.  One "step" is
one full time step of every cell of every level: mass, restriction,
halo-eta, momentum with edge rules, prolongation, halo-flux, output maxima.

* ``value`` / ``ms_per_step``: device time of exactly K steps on the
  library's stream (CUDA events bracketing ``Simulation.run(K)``, barrier +
  synchronize on both sides, max over ranks); inputs are device resident
  and 3.8 GB > 126 MB L2, so no flush is needed.
* ``e2e``: the same K steps through the public API with host buffers, as
  a fresh run: reset of the device state, one batched upload of the
  page-locked host inputs (the initial level; the bathymetry as 1-D depth
  profiles expanded on the device where it has them, else with ghosts), K steps,
  one batched download of the result maps (max_eta, max_speed,
  max_inundation: what the reference's run writes, cli.py:160-176) into
  page-locked buffers.
* ``roofline``: the momentum kernel (the dominant one), algorithmic bytes
  per launch / its average duration over the timed steps (CUDA events
  inside the graph on every 8th timed step, on the launch stream), against
  the measured HBM copy bandwidth in MEASURED_PEAKS.json; ``roofline.fp64``
  the same kernel against the measured FP64 (DFMA) rate, its binding limit.
* ``cpu_baseline``: the oracle port (oracle/, plain C + OpenMP, all host
  threads) on a bounded sample of the same workload, rank 0 only.

``--impl reference`` times the reference's CPU path (the oracle port, since
the reference is numpy code that cannot travel to the GPU box) with every
host thread on the same workload and prints the same line.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

# stdout carries exactly one JSON line: the line goes to a duplicate of the
# original stdout, and file descriptor 1 itself is pointed at stderr, so
# whatever native code prints there (NCCL's version line under torchrun on
# some boxes, even with NCCL_DEBUG_FILE set) lands on stderr
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
_JSON_OUT = None


def emit(line):
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SIX_HOURS_STEPS = 108_000
ALG_BYTES_STEP = 88.0        # B/cell-step, all-wet domain
ALG_BYTES_MOM = 48.0         # B/cell per momentum launch (eta, h, M, N read; M, N write)


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def build_workload(P, name, scale):
    if name == "kochi":
        system = P.build_kochi_scaled_config(scale)
        settings = P.kochi_settings(system)
        return system, settings, f"kochi-5level scale {scale} (BASELINE config 3)"
    sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
    import systems
    if name in ("cfg1", "cfg2"):
        system, settings, _ = systems.make(P, name)
        return system, settings, f"{name} (BASELINE config {name[-1]})"
    if name == "cfg5":
        system, settings, _ = systems.cfg5(P, scale)
        return system, settings, f"cfg5 single-level 10 m, {system.cell_count} cells in 8 strips (BASELINE config 5)"
    if name == "cfg5weak":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        system, settings, _ = systems.cfg5(P, scale, strips=world, rows=int(round(2500 * scale)))
        return system, settings, (f"cfg5 weak scaling: one {system.levels[0].blocks[0].ni} x "
                                  f"{system.levels[0].blocks[0].nj} strip per GPU (BASELINE config 5)")
    raise SystemExit(f"unknown config {name}")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device, self.proc, self.lines = device, None, []
        self.window = (0.0, float("inf"))      # host-clock bounds of the timed region

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        lo, hi = self.window
        for ts, ln in self.lines:
            if not lo <= ts <= hi:
                continue
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[5 + k].lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def profiled_traffic():
    """dram bytes/launch of the momentum kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "momentum_traffic.json")
    try:
        with open(p) as f:
            return float(json.load(f)["bytes_per_step"])
    except (OSError, ValueError, KeyError):
        return None


def fp64_roofline(cells, mom_s):
    """The momentum kernel against the FP64 pipe: its FP64 instructions per
    cell (counted by ncu, profiles/r02/march_ncu.json: sm__inst_executed_pipe_fp64
    of every march launch of one step / cells) over the event-timed launch
    duration, against the DFMA rate tools/micro/dp_pipe.cu measured on a
    B200 (profiles/r02/fp64_peak.json).  The kernel is FP64/issue bound,
    not HBM bound; this is its binding roofline."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02", "march_ncu.json")) as f:
            prof = json.load(f)
        with open(os.path.join(ROOT, "profiles", "r02", "fp64_peak.json")) as f:
            peak = json.load(f)
    except (OSError, ValueError):
        return None
    dp_per_cell = prof["dp_thread_inst_per_cell"]
    achieved = dp_per_cell * cells / mom_s if mom_s > 0 else None
    return {"bound": "fp64", "unit": "DP inst/s", "achieved": achieved, "peak": peak["dp_inst_per_s"],
            "frac": achieved / peak["dp_inst_per_s"] if achieved else None,
            "dp_inst_per_cell": dp_per_cell, "issue_inst_per_cell": prof.get("thread_inst_per_cell"),
            "source": "profiles/r02/march_ncu.json, profiles/r02/fp64_peak.json"}


def workload_config(P, system, settings, label, world):
    """The `config` dict both arms print (same workload, same plan)."""
    counts = [b.cell_count for _, b in system.all_blocks()]
    plan = P.packed_plan(system, world) if world > 1 else P.equal_cell_plan(counts, 1)
    return plan, {"workload": label, "cells": system.cell_count, "levels": len(system.levels),
                  "blocks": system.n_blocks, "dt_s": settings.dt,
                  "parallelism": f"blocks over {world} GPU(s) (packed plan, blocks per rank "
                                 f"{[len(plan.blocks_of(r)) for r in range(world)]})",
                  "l2": "state 3.8 GB >> 126 MB L2; no flush"}


def cpu_sample(system, settings, steps=2, warm=1):
    """The oracle on ``steps`` steps of the same workload, all host threads."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    oracle.build_library()
    threads = oracle.set_threads(os.cpu_count() or 1)
    sim = oracle.OracleSimulation(system, settings)
    sim.run(warm)
    t0 = time.perf_counter()
    sim.run(steps)
    dt = time.perf_counter() - t0
    return system.cell_count * steps / dt / 1e9, threads, dt


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import paper_2408_07609_b200 as P
    system, settings, label = build_workload(P, args.config, args.scale)
    _, config = workload_config(P, system, settings, label, args.gpus)
    # exactly K steps after W warm-up steps, as the GPU arm, unless that
    # would take the host more than ~4 minutes (the oracle port manages
    # ~0.06 Gcell/s on 16-24 threads: K <= ~300 at Kochi-1.0)
    budget_steps = max(1, int(240.0 * 0.06e9 / system.cell_count))
    steps = max(1, min(args.steps, budget_steps))
    warm = max(1, min(args.warmup, budget_steps // 4 + 1))
    rate, threads, dt = cpu_sample(system, settings, steps=steps, warm=warm)
    line = {
        "impl": "reference", "metric": "Gcell-updates/s", "value": rate, "unit": "Gcell/s",
        "n_gpus": args.gpus, "steps": steps, "warmup": warm, "ms_per_step": dt / steps * 1e3,
        "higher_is_better": True,
        "scaling": "weak" if (args.gpus == 1 or args.config == "cfg5weak") else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "six_hour_wall_s": dt / steps * SIX_HOURS_STEPS,
        "cpu_baseline": {"value": rate, "unit": "Gcell/s", "cores": threads, "kind": "port",
                         "sample": f"{steps} steps of the full workload after {warm} warm-up steps "
                                   "(oracle/, the C restatement of the numpy reference, OpenMP over "
                                   "blocks; the numpy reference itself is ~4x slower on the same "
                                   "cores, SURVEY.md App. D)"},
        "e2e": {"value": rate, "unit": "Gcell/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    emit(line)


def run_ours(args):
    rank, world, local = dist_env()
    import torch
    import paper_2408_07609_b200 as P
    from paper_2408_07609_b200 import distributed as D
    from paper_2408_07609_b200.runner import host_block_arrays
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist is not None:
            dist.barrier()

    system, settings, label = build_workload(P, args.config, args.scale)
    cells = system.cell_count
    counts = [b.cell_count for _, b in system.all_blocks()]
    # blocks -> GPUs: packed (not only consecutive runs) so that the mass and
    # the momentum phase are both balanced under the measured B200 per-width
    # costs (balance.packed_plan)
    plan, config = workload_config(P, system, settings, label, world)
    torch.cuda.synchronize()
    t_setup = time.perf_counter()
    # setup: host initial level (np.exp), device-built bathymetry where the
    # depth is a 1-D profile, descriptor, arena, tables
    sim = P.Simulation(system, settings, plan, device=local, distributed=world > 1)
    setup_s = time.perf_counter() - t_setup
    ext = torch.cuda.ExternalStream(sim.stream_ptr, device=local)
    sim.run(args.warmup, threaded=False)
    sim.set_timing(True)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the sampler starts ahead (nvidia-smi needs a few hundred ms) and keeps
    # only the samples read while the timed steps ran
    # clock samples: the second warm-up run and the timed run back to back
    # (the same kernels under the same load; a K = 20 timed region alone is
    # shorter than nvidia-smi's 50 ms period)
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        w0 = time.time()
        sim.run(max(args.warmup, 100), threaded=False)     # >= 0.2 s of load: several samples
        barrier()
        torch.cuda.synchronize()
        # ranks leave the host barrier up to a few hundred us apart; meeting
        # on the device right before the start event keeps that skew out of
        # the max-over-ranks time
        sim.device_barrier()
        start.record(ext)
        sim.run(args.steps, threaded=False)
        end.record(ext)
        torch.cuda.synchronize()
        clk.mark(w0, time.time())
    barrier()
    sim.set_timing(False)
    t_local = start.elapsed_time(end) / 1e3
    t = D.max_over_ranks(t_local) if world > 1 else t_local
    mass_s, mom_s, step_s = sim.kernel_seconds()
    launches = sim.launches_per_step * args.steps + 4
    my_cells = sum(c for k, c in enumerate(counts) if sim.owner[k] == rank)
    per_rank = [(rank, my_cells, mass_s, mom_s, step_s)]
    if world > 1:
        import pickle
        per_rank = [pickle.loads(b) for b in D.all_gather_bytes(pickle.dumps(per_rank[0]))]

    # end to end through the public API with host buffers, as a fresh run:
    # reset the device state, upload the host inputs (one batched transfer),
    # K steps, download the result maps (one batched transfer; every rank
    # its own blocks)
    # page-locked inputs: the initial level, and the bathymetry (its 1-D
    # depth profiles where it has them, expanded on the device: §8(f)3)
    arrays = host_block_arrays(system, settings, pinned=True, device_bathymetry=True)
    outs = sim.output_buffers(pinned=True, fields=sim.RESULT_FIELDS)
    # untimed warm-up of the transfer path (its device staging is allocated
    # on first use)
    sim.reset()
    sim.upload_initial_state(arrays)
    sim.download_outputs(outs)
    barrier()
    sim.device_barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.reset()
    h2d = sim.upload_initial_state(arrays)
    sim.run(args.steps, threaded=False)
    _, d2h = sim.download_outputs(outs)
    te_local = time.perf_counter() - t0
    te = D.max_over_ranks(te_local) if world > 1 else te_local
    if world > 1:
        h2d = sum(D.all_gather_bytes(h2d))
        d2h = sum(D.all_gather_bytes(d2h))

    peak, peak_src = measured_peaks()
    achieved = ALG_BYTES_MOM * my_cells / mom_s / 1e9 if mom_s > 0 else None
    traffic = profiled_traffic() if world == 1 else None   # the capture is of the 1-GPU step
    line = {
        "metric": "Gcell-updates/s", "value": cells * args.steps / t / 1e9, "unit": "Gcell/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak" if (world == 1 or args.config == "cfg5weak") else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config,
        "six_hour_wall_s": t / args.steps * SIX_HOURS_STEPS,
        "setup_s": setup_s,
        "step_roofline": {"bytes_per_cell_step": ALG_BYTES_STEP,
                          "achieved_gbs": ALG_BYTES_STEP * cells / (t / args.steps) / 1e9,
                          "frac": ALG_BYTES_STEP * cells / (t / args.steps) / 1e9 / (peak * world)},
        "roofline": {"kernel": "k_momentum", "bound": "hbm", "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak if achieved else None,
                     "traffic": traffic, "alg_bytes_per_launch": ALG_BYTES_MOM * my_cells,
                     "avg_launch_s": mom_s, "peak_source": peak_src,
                     "mass_kernel_s": mass_s, "step_s_events": step_s, "rank": rank,
                     "fp64": fp64_roofline(my_cells, mom_s)},
        "e2e": {"value": cells * args.steps / te / 1e9, "unit": "Gcell/s",
                "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": d2h / args.steps,
                "wall_s": te},
        "gpu_launches": launches,
        "ranks": [{"rank": r, "cells": c, "mass_s": m, "momentum_s": k, "step_s": st}
                  for r, c, m, k, st in per_rank],
        "clocks": clk.summary(),
    }
    if rank == 0 and not args.no_cpu and world == 1:
        n_cpu = max(1, int(12.0 * 0.06e9 / cells))             # ~10-15 s of host work
        rate, threads, dt = cpu_sample(system, settings, steps=n_cpu, warm=1)
        line["cpu_baseline"] = {"value": rate, "unit": "Gcell/s", "cores": threads, "kind": "port",
                                "sample": f"{n_cpu} steps of the full workload after 1 warm-up step "
                                          f"({dt:.1f} s)"}
    if rank == 0:
        emit(line)
    sim.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=("ours", "reference"))
    ap.add_argument("--config", default="kochi")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
