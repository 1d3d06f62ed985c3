"""Where Simulation() setup time goes on Kochi-1.0 (one GPU): cProfile of the
constructor, plus the library's own ts_create / merged-exchange timings
(TSUNAMI_B200_VERBOSE).

    python tools/setup_profile.py
"""
import cProfile, pstats, os, sys, time
sys.path.insert(0, os.getcwd())
os.environ["TSUNAMI_B200_VERBOSE"] = "1"
import torch
import paper_2408_07609_b200 as P
s = P.build_kochi_scaled_config(1.0)
st = P.kochi_settings(s)
torch.cuda.synchronize()
plan = P.equal_cell_plan([b.cell_count for _, b in s.all_blocks()], 1)
t = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
sim = P.Simulation(s, st, plan, device=0, distributed=False)
pr.disable()
print("setup", time.perf_counter() - t)
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
