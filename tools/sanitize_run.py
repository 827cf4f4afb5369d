"""Small runs of every evolve kernel family for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck), SURVEY §5:

    compute-sanitizer --tool racecheck python tools/sanitize_run.py

TSP (static + NVRTC with user operators, crossover snapshots, deferred
whole-row operators), QAP, knapsack, JSP-int, VRPTW, a user problem with a
user operator, and a MULTI_FIXED user problem — full reference registries."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2603_19163_b200 as G  # noqa: E402
from paper_2603_19163_b200 import instances as I  # noqa: E402

cfg = dict(population=6, team_size=32, max_generations=12, seed=3, device_init=True)
d = I.tsp_random(40, 5)
runs = {
    "tsp": G.builtin_problem("tsp", G.InstanceData(distance_matrix=d)),
    "qap": G.builtin_problem("qap", G.InstanceData(flow_matrix=I.qap_random(20, 3)[0],
                                                   distance_matrix=I.qap_random(20, 3)[1])),
    "knap": G.builtin_problem("knapsack", G.InstanceData(
        weights=I.knapsack_random(100, 4)[0], values=I.knapsack_random(100, 4)[1],
        capacity=I.knapsack_random(100, 4)[2])),
    "jsp": G.builtin_problem("jsp_int", G.InstanceData(jobs=I.jsp_random(5, 4, 9))),
}
vd = I.vrptw_solomon_like(n=20, vehicles=5, seed=7)
runs["vrptw"] = G.builtin_problem("vrptw", G.InstanceData(
    distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity, vehicles=vd.vehicles,
    ready_times=vd.ready, due_times=vd.due, service_times=vd.service))
runs["jsp_perm"] = G.builtin_problem("jsp_perm", G.InstanceData(jobs=I.jsp_random(5, 4, 11)))
runs["vrp_priority"] = G.builtin_problem("vrp_priority", G.InstanceData(
    distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity, vehicles=vd.vehicles,
    priorities=np.arange(20) % 3))
runs["cvrp_lex"] = G.builtin_problem("cvrp", G.InstanceData(
    distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity, vehicles=vd.vehicles,
    meta={"objectives": ("distance", "vehicles"),
          "comparison": G.Lexicographic((1, 0), (0.0, 0.0))}))
runs["schedule"] = G.builtin_problem("schedule_binary", G.InstanceData(
    cost_matrix=np.arange(24.0).reshape(6, 4) % 7 + 1, requirements=np.array([2.0, 1, 3, 1])))
# guided-rebuild / crossover dominated registries (the rare whole-row paths)
GR_HEAVY = {"tsp": (16, 12, 0), "qap": (16, 12), "knap": (16, 13), "jsp": (16, 13),
            "vrptw": (16, 12, 9), "vrp_priority": (16, 15, 10), "jsp_perm": (16, 12, 15),
            "schedule": (16, 13, 6)}
for name, ops in GR_HEAVY.items():
    prob = runs[name]
    prob.device_sequences = (lambda o: lambda: o)(ops)
    r = G.run(prob, G.EngineConfig(population=4, team_size=32, max_generations=4, seed=5,
                                   islands=G.IslandsConfig(count=2, migration="hybrid",
                                                           interval=2)))
    print(f"{name} GR-heavy {ops}: {r.objectives} err {r.device.get('error_flags')}", flush=True)
for name, prob in runs.items():
    if name in GR_HEAVY:
        del prob.device_sequences  # back to the class's full registry
for name, prob in runs.items():
    ops = G.tsp_delta_operators() if name == "tsp" else ()
    r = G.run(prob, G.EngineConfig(custom_operators=ops, **cfg))
    print(f"{name}: {r.objectives} pen {r.penalty} gens {r.generations_completed} "
          f"err {r.device.get('error_flags')}", flush=True)
TOUR = """
  double s = 0.0;
  for (int i = 0; i < sol.n; ++i) s += data.dist[sol[i] * sol.n + sol[i + 1 == sol.n ? 0 : i + 1]];
  return s;
"""
KICK = """
  const int i = ctx.randbelow(ctx.n), j = ctx.randbelow(ctx.n);
  if (i != j) ctx.swap(i, j);
"""
r = G.solve_custom(encoding="permutation", dim2=40, compute_obj=TOUR, data={"dist": d},
                   custom_operators=[G.CustomOperator(100, "kick", cuda=KICK)], time_limit=None,
                   **cfg)
print(f"user: {r.objectives} gens {r.generations_completed}", flush=True)
# long rows in global memory (row layouts 12 / 13), single-team CTAs
w, v, cap = I.knapsack_random(6000, 77)
r = G.run(G.builtin_problem("knapsack", G.InstanceData(weights=w, values=v, capacity=cap)),
          G.EngineConfig(population=3, team_size=64, max_generations=4, seed=3))
print(f"knap6000: layout {r.device['layout']} {r.objectives}", flush=True)
r = G.run(G.CudaProblem("permutation", 40, TOUR, data={"dist": d}),
          G.EngineConfig(population=2, team_size=32, teams_per_cta=1, max_generations=6, seed=1))
print(f"single-team CTA: {r.objectives}", flush=True)
# two objectives, Lexicographic with a Maximize objective
ASC = "int k = 0; for (int i = 0; i + 1 < sol.n; ++i) k += sol[i] < sol[i + 1]; return (double)k;"
prob2 = G.CudaProblem("permutation", 40, [TOUR, ASC], data={"dist": d}, maximize=(False, True),
                      comparison=G.Lexicographic((1, 0), (0.0, 2.0)))
r = G.run(prob2, G.EngineConfig(population=4, team_size=32, max_generations=6, seed=2,
                                islands=G.IslandsConfig(count=2, migration="hybrid", interval=2)))
print(f"two-objective lex: {r.objectives}", flush=True)
print("sanitize_run done")
