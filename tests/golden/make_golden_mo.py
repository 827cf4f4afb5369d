"""Multi-objective golden runs from the UNMODIFIED reference (build container only).

    PYTHONPATH=/root/repo python tests/golden/make_golden_mo.py

Bi-objective routing (builtins.py:80-152 objectives ("distance", "vehicles")) with
Weighted and Lexicographic comparisons (core.py:80-106, :315-347, engine.py:225-246)
and non-dominated-sort initialisation (engine.py:352-420).  Instances: the
reference's own eight-customer fixture (instances.py:170-184) and a 30-customer
synthetic VRPTW.  Writes tests/golden/golden_mo.json.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

REF = "/root/reference/pkg/src"
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
sys.path.insert(0, REF)  # the reference genopt wins over the repo's drop-in shim

import genopt as G  # noqa: E402
from genopt import instances as GI  # noqa: E402
from genopt.core import Lexicographic, Weighted  # noqa: E402

from paper_2603_19163_b200 import instances as I  # noqa: E402

OUT = Path(__file__).with_name("golden_mo.json")

CASES = {
    # key: (instance, objectives, comparison spec, P, T, G, seed, islands)
    "cvrp8_w": ("cvrp8", ("distance", "vehicles"), None, 6, 16, 40, 42, 1),
    "cvrp8_w100": ("cvrp8", ("distance", "vehicles"), ("w", (1.0, 100.0)), 6, 16, 40, 7, 1),
    "cvrp8_lex_veh": ("cvrp8", ("distance", "vehicles"), ("lex", (1, 0), (0.0, 0.0)), 6, 16, 40,
                      123, 1),
    "cvrp8_lex_tol": ("cvrp8", ("distance", "vehicles"), ("lex", (0, 1), (10.0, 0.0)), 6, 16, 40,
                      99, 1),
    "vrptw30_w": ("vrptw30", ("distance", "vehicles"), ("w", (1.0, 50.0)), 4, 16, 15, 5, 1),
    "vrptw30_lex": ("vrptw30", ("distance", "vehicles"), ("lex", (1, 0), (0.0, 0.0)), 6, 16, 20,
                    11, 2),
}


def comparison(spec):
    if spec is None:
        return None
    if spec[0] == "w":
        return Weighted(spec[1])
    return Lexicographic(spec[1], spec[2])


def instance(name, objectives, comp):
    if name == "cvrp8":
        data = GI.cvrp8_instance(objectives=objectives, comparison=comp)
        return G.builtin_problem("cvrp", data), {
            "dist": data.distance_matrix.tolist(), "demands": list(map(float, data.demands)),
            "capacity": float(data.capacity), "vehicles": int(data.vehicles), "tw": False}
    vd = I.vrptw_solomon_like(n=30, vehicles=6, seed=7)
    meta = {"objectives": objectives}
    if comp is not None:
        meta["comparison"] = comp
    data = G.InstanceData(distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity,
                          vehicles=vd.vehicles, ready_times=vd.ready, due_times=vd.due,
                          service_times=vd.service, meta=meta)
    return G.builtin_problem("vrptw", data), {"vrptw_solomon_like": [30, 6, 7], "tw": True}


def main():
    out = {"generator": "tests/golden/make_golden_mo.py", "runs": {}}
    for key, (name, objs, cspec, P, T, Gn, seed, isl) in CASES.items():
        comp = comparison(cspec)
        prob, inst = instance(name, objs, comp)
        cfg = G.EngineConfig(population=P, team_size=T, max_generations=Gn, seed=seed,
                             record_history=True,
                             islands=G.IslandsConfig(count=isl, migration="hybrid", interval=5))
        r = G.run(prob, cfg)
        out["runs"][key] = {
            "instance": inst, "objectives_names": list(objs), "comparison": cspec,
            "config": {"population": P, "team_size": T, "max_generations": Gn, "seed": seed,
                       "islands": isl},
            "best": {"data": [[int(x) for x in r.best.row(rr)] for rr in range(r.best.d1)]},
            "objectives": [float(x) for x in r.objectives], "penalty": float(r.penalty),
            "history": r.history["best_phi"], "generations": r.generations_completed,
            "weights": [float(e["weight"]) for e in r.final_weights["sequences"]],
            "ids": [e["id"] for e in r.final_weights["sequences"]],
            "k_weights": list(r.final_weights["k_steps"]),
        }
        print(key, r.objectives, r.penalty, flush=True)
    OUT.write_text(json.dumps(out))


if __name__ == "__main__":
    main()
