"""Reference results for the equal-budget gap-parity tests on the benchmark
shapes (build container only; VERDICT r1 "Next" #2):

    PYTHONPATH=/root/repo python tests/golden/make_gap_golden_bench.py [case ...]

Runs the UNMODIFIED reference `genopt.run()` (/root/reference/pkg/src, never
shipped) for the ten engine seeds of SURVEY §8(d) at a fixed evaluation
budget, one process per run:
  * c2      — the pcb442-shaped lattice (C2) with the tsp-delta user operators,
              P=32 evolvers x T=128 lanes x G=200 generations
  * r101    — VRPTW on the reference's R101 fixture (C3), P=16 x T=64 x G=150
Writes tests/golden/gap_bench.json:
{cases: {name: {config...}}, seeds: [...], runs: {name: {seed: [objective, penalty]}}}.
"""

from __future__ import annotations

import json
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

REF = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).with_name("gap_bench.json")
SEEDS = (42, 123, 456, 789, 2024, 7, 99, 314, 2718, 31337)
CASES = {
    "c2": {"workload": "C2", "population": 32, "team_size": 128, "max_generations": 200},
    "r101": {"workload": "C3", "population": 16, "team_size": 64, "max_generations": 150},
}


def one(args):
    name, seed = args
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, REF)  # the reference genopt wins over the repo's drop-in shim
    import genopt as G
    from genopt import demo_ops

    from paper_2603_19163_b200 import instances as I
    c = CASES[name]
    kind, inst, _ = I.baseline_instances()[c["workload"]]
    fields = {k: v for k, v in vars(inst).items() if v is not None and k != "meta"}
    prob = G.builtin_problem(kind, G.InstanceData(**fields))
    ops = list(demo_ops.tsp_delta_operators()) if c["workload"] == "C2" else []
    cfg = G.EngineConfig(population=c["population"], team_size=c["team_size"],
                         max_generations=c["max_generations"], seed=seed, custom_operators=ops)
    res = G.run(prob, cfg)
    return name, seed, [float(res.objectives[0]), float(res.penalty)]


def main():
    names = sys.argv[1:] or list(CASES)
    data = json.loads(OUT.read_text()) if OUT.exists() else {"cases": {}, "runs": {}}
    data["seeds"] = list(SEEDS)
    jobs = [(n, s) for n in names for s in SEEDS]
    with ProcessPoolExecutor(max_workers=8) as ex:
        for name, seed, res in ex.map(one, jobs):
            data["cases"][name] = CASES[name]
            data["runs"].setdefault(name, {})[str(seed)] = res
            print(name, seed, res, flush=True)
            OUT.write_text(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
