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
print("sanitize_run done")
