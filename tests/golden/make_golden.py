"""Freeze golden vectors from the UNMODIFIED reference (build container only).

    PYTHONPATH=/root/repo python tests/golden/make_golden.py

Imports `genopt` from /root/reference/pkg/src (read-only, never shipped) and
writes tests/golden/golden.json.  Everything the oracle is pinned against
comes from here: objective values at the BASELINE shapes, operator outputs
under seeded MT19937 draws, AOS updates, population sizing, stream hashes and
whole-run trajectories (best genes, objectives, history, final weights).
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
from genopt import aos as GA  # noqa: E402
from genopt import demo_ops, operators as GO  # noqa: E402
from genopt.engine import (EngineConfig, IslandsConfig, adaptive_population_size,  # noqa: E402
                           mix64, random_solution)

from paper_2603_19163_b200 import instances as I  # noqa: E402

OUT = Path(__file__).with_name("golden.json")


def problems():
    d51 = I.tsp_random(51, 51, True)
    d51f = I.tsp_random(51, 51, False)
    d442, _ = I.tsp_lattice()
    vd = I.vrptw_solomon_like()
    f, dq = I.qap_random(100, 100)
    jobs = I.jsp_random(20, 15, 2015)
    w, v, cap = I.knapsack_random(1000, 1000)
    return {
        "tsp51": G.builtin_problem("tsp", G.InstanceData(distance_matrix=d51)),
        "tsp51f": G.builtin_problem("tsp", G.InstanceData(distance_matrix=d51f)),
        "tsp442": G.builtin_problem("tsp", G.InstanceData(distance_matrix=d442)),
        "vrptw100": G.builtin_problem("vrptw", G.InstanceData(
            distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity,
            vehicles=vd.vehicles, ready_times=vd.ready, due_times=vd.due,
            service_times=vd.service)),
        "qap100": G.builtin_problem("qap", G.InstanceData(flow_matrix=f, distance_matrix=dq)),
        "jsp20x15": G.builtin_problem("jsp_int", G.InstanceData(jobs=jobs)),
        "knap1000": G.builtin_problem("knapsack", G.InstanceData(weights=w, values=v,
                                                                 capacity=cap)),
    }


def sol_json(s):
    return {"data": [[int(x) for x in s.row(r)] for r in range(s.d1)]}


def main():
    out = {"generator": "tests/golden/make_golden.py", "reference": REF}
    probs = problems()

    # 1. objective / penalty at the BASELINE shapes
    evals = {}
    for name, p in probs.items():
        cfg = p.config()
        rows = []
        for k in range(6):
            s = random_solution(cfg, random.Random(1000 + k))
            obj, pen = G.evaluate(p, s)
            rows.append({**sol_json(s), "obj": [float(o) for o in obj], "pen": float(pen)})
        evals[name] = rows
    out["evaluate"] = evals

    # 2. operator outputs under seeded MT draws
    ops = {}
    cases = [("tsp51", [0, 1, 2, 3, 4, 14, 15]), ("vrptw100", [0, 1, 2, 3, 9, 10, 11, 15]),
             ("jsp20x15", [7, 8, 15]), ("knap1000", [5, 6, 15]), ("qap100", [0, 1, 2, 3])]
    fns = {sid: fn for sid, _, fn in GO._BUILTIN_DEFS}
    for name, ids in cases:
        p = probs[name]
        cfg = p.config()
        for sid in ids:
            rows = []
            for k in range(4):
                s = random_solution(cfg, random.Random(77 + k))
                before = sol_json(s)
                fns[sid](s, random.Random(500 + 31 * sid + k), GO.OperatorContext(p, cfg))
                rows.append({"before": before, "rng_seed": 500 + 31 * sid + k, "after": sol_json(s)})
            ops[f"{name}:{sid}"] = rows
    p = probs["tsp51"]
    for op in demo_ops.tsp_delta_operators():
        rows = []
        for k in range(4):
            s = random_solution(p.config(), random.Random(90 + k))
            before = sol_json(s)
            op.apply(s, random.Random(700 + op.id + k), GO.OperatorContext(p, p.config()))
            rows.append({"before": before, "rng_seed": 700 + op.id + k, "after": sol_json(s)})
        ops[f"tsp51:{op.id}"] = rows
    out["operators"] = ops

    # 3. AOS updates (fuzzed counters) and sampling
    rng = random.Random(4242)
    aos_rows = []
    for _ in range(40):
        nseq = rng.randrange(2, 12)
        caps = [rng.choice([float("inf"), 0.005, 0.02, 0.3]) for _ in range(nseq)]
        ws = [rng.uniform(0.01, 1.0) for _ in range(nseq)]
        entries = [GO.SequenceEntry(i, f"s{i}", None, weight=w, cap=c)
                   for i, (w, c) in enumerate(zip(ws, caps))]
        reg = GO.SequenceRegistry(entries)
        init = [e.weight for e in reg.entries]
        usage = [rng.randrange(0, 500) for _ in range(nseq)]
        impr = [rng.randrange(0, u + 1) for u in usage]
        stats = GA.AosStats(reg.ids())
        stats.usage[:] = usage
        stats.improvement[:] = impr
        GA.update_weights(reg, stats, GA.AosConfig())
        first = [float(e.weight) for e in reg.entries]
        stats.usage[:] = usage[::-1]
        stats.improvement[:] = [min(a, b) for a, b in zip(impr[::-1], usage[::-1])]
        GA.update_weights(reg, stats, GA.AosConfig())
        second = [float(e.weight) for e in reg.entries]
        kw = GA.update_k_weights(GA.DEFAULT_K_WEIGHTS, usage[:3] + [0] * (3 - len(usage[:3])),
                                 impr[:3] + [0] * (3 - len(impr[:3])), GA.AosConfig())
        draws = [GA.sample_sequence(reg, random.Random(9000 + j)) for j in range(16)]
        aos_rows.append({"weights": ws, "caps": [None if c == float("inf") else c for c in caps],
                         "normalized": init, "usage": usage, "impr": impr, "first": first,
                         "second": second, "k": list(kw), "draws": draws})
    out["aos"] = aos_rows

    # 4. population sizing and stream hashes
    rng = random.Random(12)
    sizing = []
    for _ in range(200):
        args = (rng.randrange(1, 300), rng.randrange(1, 10 ** 8), rng.randrange(1, 10 ** 7),
                rng.randrange(1, 10 ** 6))
        sizing.append([*args, adaptive_population_size(*args)])
    sizing.append([108, 40 * 1024 * 1024, 763 * 1024, 96 * 1024,
                   adaptive_population_size(108, 40 * 1024 * 1024, 763 * 1024, 96 * 1024)])
    out["sizing"] = sizing
    out["mix64"] = [[list(parts), mix64(*parts)] for parts in
                    [(42,), (42, 0, 1, 0, 0), (42, 7, 99, 127, 0), (2024, 3, 1, 0, 1),
                     (123, 2), (456, 4, 101), (2 ** 63, 2 ** 64 - 1, 5)]]

    # 5. whole-run trajectories (the oracle engine must reproduce these)
    runs = {}

    def record(key, p, **kw):
        islands = kw.pop("islands", IslandsConfig())
        cfg = EngineConfig(record_history=True, islands=islands, **kw)
        r = G.run(p, cfg)
        runs[key] = {
            "config": {**{k: (v if not isinstance(v, tuple) else None) for k, v in kw.items()
                          if k != "custom_operators"},
                       "custom": bool(kw.get("custom_operators")),
                       "islands": islands.as_dict()},
            "best": sol_json(r.best), "objectives": r.objectives, "penalty": r.penalty,
            "history": r.history["best_phi"], "generations": r.generations_completed,
            "weights": [float(e["weight"]) for e in r.final_weights["sequences"]],
            "ids": [e["id"] for e in r.final_weights["sequences"]],
            "k_weights": list(r.final_weights["k_steps"]),
        }

    record("tsp51", probs["tsp51"], population=8, team_size=16, max_generations=60, seed=42)
    record("tsp51_delta", probs["tsp51"], population=8, team_size=16, max_generations=40,
           seed=123, custom_operators=demo_ops.tsp_delta_operators(),
           islands=IslandsConfig(count=2, migration="hybrid", interval=20))
    record("tsp51f", probs["tsp51f"], population=6, team_size=16, max_generations=40, seed=7)
    record("qap100", probs["qap100"], population=4, team_size=8, max_generations=12, seed=456)
    record("jsp20x15", probs["jsp20x15"], population=4, team_size=8, max_generations=6, seed=789)
    record("knap1000", probs["knap1000"], population=4, team_size=8, max_generations=12, seed=2024)
    record("vrptw100", probs["vrptw100"], population=4, team_size=8, max_generations=4, seed=42,
           islands=IslandsConfig(count=2, migration="ring", interval=2),
           elite_injection_interval=3)
    out["runs"] = runs
    OUT.write_text(json.dumps(out, separators=(",", ":")))
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
