"""Reference results for the row-family gap-parity tests (build container only).

    PYTHONPATH=/root/repo python tests/golden/make_gap_golden_rows.py

Runs the UNMODIFIED reference `genopt.run()` (/root/reference/pkg/src) with its
full built-in registry on small instances of the row-kernel BASELINE families
— QAP (permutation, n=30), 0/1 knapsack (binary, n=200), JSP-int (integer,
6 jobs x 5 machines) — for ten engine seeds at a fixed evaluation budget, one
process per run.  Writes tests/golden/gap_rows.json.
"""

from __future__ import annotations

import json
import sys
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

REF = "/root/reference/pkg/src"
ROOT = Path(__file__).resolve().parents[2]
OUT = Path(__file__).with_name("gap_rows.json")
SEEDS = (42, 123, 456, 789, 2024, 7, 99, 314, 2718, 31337)
CASES = {
    "qap30": {"population": 8, "team_size": 32, "max_generations": 120},
    "knap200": {"population": 8, "team_size": 32, "max_generations": 150},
    "jsp6x5": {"population": 8, "team_size": 32, "max_generations": 100},
}


def instance(name):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, REF)  # the reference genopt wins over the repo's drop-in shim
    import genopt as G

    from paper_2603_19163_b200 import instances as I
    if name == "qap30":
        f, d = I.qap_random(30, 100)
        return G.builtin_problem("qap", G.InstanceData(flow_matrix=f, distance_matrix=d))
    if name == "knap200":
        w, v, cap = I.knapsack_random(200, 1000)
        return G.builtin_problem("knapsack", G.InstanceData(weights=w, values=v, capacity=cap))
    return G.builtin_problem("jsp_int", G.InstanceData(jobs=I.jsp_random(6, 5, 7)))


def one(args):
    name, seed = args
    prob = instance(name)
    from genopt import EngineConfig, run
    c = CASES[name]
    res = run(prob, EngineConfig(population=c["population"], team_size=c["team_size"],
                                 max_generations=c["max_generations"], seed=seed))
    return name, seed, float(res.objectives[0]), float(res.penalty)


def main():
    jobs = [(n, s) for n in CASES for s in SEEDS]
    runs = {n: {} for n in CASES}
    with ProcessPoolExecutor(max_workers=8) as ex:
        for name, seed, best, pen in ex.map(one, jobs):
            runs[name][str(seed)] = [best, pen]
            print(name, seed, best, pen, flush=True)
    OUT.write_text(json.dumps({"cases": CASES, "seeds": list(SEEDS), "runs": runs}, indent=1))


if __name__ == "__main__":
    main()
