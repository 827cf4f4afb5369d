"""Reference results for the equal-budget gap-parity test (build container only).

    PYTHONPATH=/root/repo python tests/golden/make_gap_golden.py

Runs the UNMODIFIED reference `genopt.run()` (/root/reference/pkg/src, never
shipped) on the C1 shape (random Euclidean TSP n=51, TSPLIB nint distances,
instance seed 51) for the ten engine seeds of SURVEY §8(d) at a fixed
evaluation budget (P=16 evolvers x T=32 lanes x G generations), with the full
built-in registry, and with the user-registered tsp-delta operators on top.
One process per seed.  Writes tests/golden/gap_c1.json:
{config: {...}, runs: {"builtin": {seed: best}, "tsp_delta": {seed: best}}}.
"""

from __future__ import annotations

import json
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

REF = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).with_name("gap_c1.json")
SEEDS = (42, 123, 456, 789, 2024, 7, 99, 314, 2718, 31337)
CFG = {"population": 16, "team_size": 32, "max_generations": 300, "instance": "tsp_random(51, 51)"}


def one(args):
    variant, seed = args
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, REF)  # the reference genopt wins over the repo's drop-in shim
    import genopt as G
    from genopt import demo_ops

    from paper_2603_19163_b200 import instances as I
    d = I.tsp_random(51, 51, True)
    prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=d))
    ops = list(demo_ops.tsp_delta_operators()) if variant == "tsp_delta" else []
    cfg = G.EngineConfig(population=CFG["population"], team_size=CFG["team_size"],
                         max_generations=CFG["max_generations"], seed=seed, custom_operators=ops)
    res = G.run(prob, cfg)
    return variant, seed, float(res.objectives[0])


def main():
    jobs = [(v, s) for v in ("builtin", "tsp_delta") for s in SEEDS]
    runs = {"builtin": {}, "tsp_delta": {}}
    with ProcessPoolExecutor(max_workers=8) as ex:
        for variant, seed, best in ex.map(one, jobs):
            runs[variant][str(seed)] = best
            print(variant, seed, best, flush=True)
    OUT.write_text(json.dumps({"config": CFG, "seeds": list(SEEDS), "runs": runs}, indent=1))


if __name__ == "__main__":
    main()
