"""Kernel timing of one library build on the Kochi-shaped workload.

    TSUNAMI_B200_LIB=variants/x.so python tools/kbench.py [--scale 1.0] [--steps 60]
"""
import argparse, json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2408_07609_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=1.0)
ap.add_argument("--steps", type=int, default=60)
ap.add_argument("--tile-rows", type=int, default=0)
ap.add_argument("--warm", type=int, default=5)
a = ap.parse_args()
system = P.build_kochi_scaled_config(a.scale)
settings = P.kochi_settings(system)
sim = P.Simulation(system, settings, tile_rows=a.tile_rows)
sim.run(a.warm, threaded=False)
sim.set_timing(True)
sim.run(a.steps, threaded=False)
m, k, s = sim.kernel_seconds()
cells = system.cell_count
print(json.dumps({"lib": os.environ.get("TSUNAMI_B200_LIB", "default"), "T": a.tile_rows, "warm": a.warm,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("TSUNAMI_B200_")}, "mass_ms": m * 1e3,
                  "momentum_ms": k * 1e3, "step_ms": s * 1e3, "gcells": cells / s / 1e9}))
