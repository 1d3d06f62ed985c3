"""Per-run overhead of Simulation.run on Kochi-1.0: device-timed runs of
1, 2, 4, 20 and 200 steps (max over ranks), whose intercept is the run's fixed
cost (end-of-run maxima fold, error agreement, rank skew).

    python tools/run_overhead.py
    torchrun --nproc-per-node 4 --master-addr 127.0.0.1 tools/run_overhead.py
"""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2408_07609_b200 as P
from paper_2408_07609_b200 import distributed as D
local = int(os.environ.get("LOCAL_RANK", "0")); world = int(os.environ.get("WORLD_SIZE", "1"))
torch.cuda.set_device(local)
dist = None
if world > 1:
    import torch.distributed as dist
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
s = P.build_kochi_scaled_config(1.0); st = P.kochi_settings(s)
plan = P.packed_plan(s, world) if world > 1 else P.equal_cell_plan([b.cell_count for _, b in s.all_blocks()], 1)
sim = P.Simulation(s, st, plan, device=local, distributed=world > 1)
ext = torch.cuda.ExternalStream(sim.stream_ptr, device=local)
sim.run(5, threaded=False)
timing = os.environ.get("TIMING", "0") == "1"
sim.set_timing(timing)
res = {}
for K in (1, 2, 4, 20, 200, 20, 1):
    if dist: dist.barrier()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(ext)
    sim.run(K, threaded=False)
    b.record(ext)
    torch.cuda.synchronize()
    th = time.perf_counter() - t0
    te = a.elapsed_time(b) / 1e3
    if world > 1:
        te = D.max_over_ranks(te); th = D.max_over_ranks(th)
    res.setdefault(K, []).append((round(te * 1e3, 3), round(th * 1e3, 3)))
if sim.rank == 0:
    print(json.dumps({"world": world, "timing": timing, "ms (event, host) per run": res}))
sim.close()
if dist:
    dist.barrier(); dist.destroy_process_group()
