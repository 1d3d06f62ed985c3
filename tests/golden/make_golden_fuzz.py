"""Golden digests of the REFERENCE on random nested systems
(systems.random_nested): 2-3 levels, guillotine-split siblings, children
touching the parent level's edge, straddling seams and abutting each other,
wet/dry fronts, zero / scalar / per-cell Manning, random edge kinds, 1-3
ranks.  The reference runs unmodified from /root/reference/pkg/src through
its own Simulation API with the oracle's cube root swapped in for np.cbrt
(the cbrt-aligned mode of make_golden.py).  Output: fuzz.json (sha digests
of every state array incl. ghosts and the three maxima after n steps, or
the NumericsError message).

    python tests/golden/make_golden_fuzz.py [--seeds 24]
"""

import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import make_golden as MG                                    # noqa: E402  (sets up sys.path)
import systems                                              # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=24)
    args = ap.parse_args()
    MG.oracle.build_library()
    out = {}
    for seed in range(args.seeds):
        system, settings, n, nr = systems.random_nested(MG.T, seed)
        rep = MG.T.validate_system(system, settings)
        assert not rep.violations, (seed, rep.violations)
        d = {"steps": n, "ranks": nr, "cells": sum(b.cell_count for _, b in system.all_blocks()),
             "blocks": [len(lvl.blocks) for lvl in system.levels]}
        try:
            sim = MG.run_ref(system, settings, n, nr)
            d["digests"] = {k: systems.digest(v) for k, v in MG.state_arrays(sim).items()
                            if not k.endswith("/wet")}
            d["error"] = None
        except MG.K.NumericsError as exc:
            d["error"] = str(exc)
        out[str(seed)] = d
        print(seed, d["blocks"], d["cells"], nr, d["error"], flush=True)
    with open(os.path.join(HERE, "fuzz.json"), "w") as f:
        json.dump(out, f, separators=(",", ":"))


if __name__ == "__main__":
    main()
