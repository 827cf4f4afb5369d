"""Goldens for the further built-ins (assignment, graph colouring, bin packing,
load balancing, priority / nonlinear VRP, job-shop permutation rows, binary
schedule; builtins.py:193-545) from the UNMODIFIED reference (build container
only).

    PYTHONPATH=/root/repo python tests/golden/make_golden_extra.py

Writes tests/golden/golden_extra.json: instances, objective / penalty of
seeded random solutions, and small whole-run trajectories (best, history,
final weights) that the oracle must reproduce in MT mode.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, REF)  # the reference genopt wins over the repo's drop-in shim

import genopt as G  # noqa: E402
from genopt.engine import random_solution  # noqa: E402

OUT = Path(__file__).with_name("golden_extra.json")


def instances():
    rng = np.random.default_rng(77)
    n = 40
    pts = rng.integers(0, 40, size=(60, 2))
    edges = sorted({(int(min(a, b)), int(max(a, b))) for a, b in pts if a != b})
    return {
        "assign40": ("assignment", {"cost_matrix": rng.integers(1, 100, size=(n, n)).tolist()}),
        "color40": ("graph_coloring", {"edges": edges, "num_colors": 4,
                                       "meta": {"num_vertices": 40}}),
        "binpack30": ("bin_packing", {"item_sizes": rng.integers(2, 9, size=30).tolist(),
                                      "bin_capacity": 10.0}),
        "loadbal40": ("load_balancing", {"durations": rng.integers(1, 30, size=40).tolist(),
                                         "num_machines": 5}),
        "vrpprio20": ("vrp_priority", routing(rng, 20, 5, priorities=True)),
        "vrpnl20": ("vrp_nonlinear", routing(rng, 20, 5)),
        "jspperm6x4": ("jsp_perm", {"jobs": [[[int(m), int(rng.integers(1, 20))]
                                              for m in rng.permutation(4)] for _ in range(6)]}),
        "sched8x6": ("schedule_binary", {"cost_matrix": rng.integers(1, 20, size=(8, 6)).tolist(),
                                         "requirements": rng.integers(1, 4, size=6).tolist()}),
    }


def routing(rng, n, vehicles, priorities=False):
    pts = rng.uniform(0, 100, size=(n + 1, 2))
    d = np.rint(np.sqrt(((pts[:, None, :] - pts[None, :, :]) ** 2).sum(-1)))
    out = {"distance_matrix": d.tolist(), "demands": rng.integers(1, 10, size=n).tolist(),
           "capacity": 30.0, "vehicles": vehicles}
    if priorities:
        out["priorities"] = rng.integers(0, 3, size=n).tolist()
    return out


def build(name, payload):
    kw = dict(payload)
    meta = kw.pop("meta", {})
    for k in ("cost_matrix", "item_sizes", "durations", "distance_matrix", "demands", "priorities",
              "requirements"):
        if k in kw:
            kw[k] = np.asarray(kw[k], dtype=np.float64)
    if "jobs" in kw:
        kw["jobs"] = [[tuple(op) for op in ops] for ops in kw["jobs"]]
    return G.builtin_problem(name, G.InstanceData(meta=meta, **kw))


def main():
    out = {"generator": "tests/golden/make_golden_extra.py", "instances": {}, "evaluate": {},
           "runs": {}}
    for key, (name, payload) in instances().items():
        out["instances"][key] = {"problem": name, "payload": payload}
        p = build(name, payload)
        rows = []
        for k in range(8):
            s = random_solution(p.config(), random.Random(500 + k))
            obj, pen = G.evaluate(p, s)
            rows.append({"data": [[int(x) for x in s.row(r)] for r in range(s.d1)],
                         "obj": [float(o) for o in obj], "pen": float(pen)})
        out["evaluate"][key] = rows
        r = G.run(p, G.EngineConfig(population=6, team_size=16, max_generations=25, seed=11,
                                    record_history=True))
        out["runs"][key] = {
            "config": {"population": 6, "team_size": 16, "max_generations": 25, "seed": 11},
            "best": {"data": [[int(x) for x in r.best.row(q)] for q in range(r.best.d1)]},
            "objectives": [float(x) for x in r.objectives], "penalty": float(r.penalty),
            "history": r.history["best_phi"],
            "weights": [float(e["weight"]) for e in r.final_weights["sequences"]],
            "ids": [e["id"] for e in r.final_weights["sequences"]],
            "k_weights": list(r.final_weights["k_steps"]),
        }
        print(key, r.objectives, r.penalty, flush=True)
    OUT.write_text(json.dumps(out))


if __name__ == "__main__":
    main()
