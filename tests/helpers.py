"""Shared test helpers: the BASELINE-shape instances as oracle problems."""

from __future__ import annotations

import numpy as np

from oracle import problems as P
from paper_2603_19163_b200 import instances as I


def instance_arrays():
    d51 = I.tsp_random(51, 51, True)
    d51f = I.tsp_random(51, 51, False)
    d442, _ = I.tsp_lattice()
    vd = I.vrptw_solomon_like()
    f, dq = I.qap_random(100, 100)
    jobs = I.jsp_random(20, 15, 2015)
    w, v, cap = I.knapsack_random(1000, 1000)
    return dict(d51=d51, d51f=d51f, d442=d442, vd=vd, f=f, dq=dq, jobs=jobs, w=w, v=v, cap=cap)


def oracle_problems():
    a = instance_arrays()
    vd = a["vd"]
    return {
        "tsp51": P.Tsp(a["d51"]),
        "tsp51f": P.Tsp(a["d51f"]),
        "tsp442": P.Tsp(a["d442"]),
        "vrptw100": P.Vrptw(vd.dist, vd.demands, vd.capacity, vd.vehicles, vd.ready, vd.due,
                            vd.service),
        "qap100": P.Qap(a["f"], a["dq"]),
        "jsp20x15": P.JspInt(a["jobs"]),
        "knap1000": P.Knapsack(a["w"], a["v"], a["cap"]),
    }


def sol_from_json(problem, js):
    spec = problem.spec
    data = np.zeros((spec.d1, spec.d2), dtype=np.int64)
    sizes = np.zeros(spec.d1, dtype=np.int64)
    for r, row in enumerate(js["data"]):
        data[r, :len(row)] = row
        sizes[r] = len(row)
    return P.Sol(data, sizes, spec.m)


def sol_rows(sol):
    return [[int(x) for x in sol.row(r)] for r in range(sol.d1)]


def bench_pairs(names=("C1", "C2", "C3", "C4", "C5a", "C5b")):
    """The BASELINE workloads as (device problem, oracle problem, custom ops):
    instances.baseline_instances(), C2 with the tsp-delta user operators."""
    import paper_2603_19163_b200 as G
    from oracle import moves as M
    out = {}
    table = I.baseline_instances()
    for name in names:
        kind, inst, _ = table[name]
        prob = G.builtin_problem(kind, inst)
        if kind == "tsp":
            ref = P.Tsp(inst.distance_matrix)
        elif kind == "vrptw":
            ref = P.Vrptw(inst.distance_matrix, inst.demands, inst.capacity, inst.vehicles,
                          inst.ready_times, inst.due_times, inst.service_times)
        elif kind == "qap":
            ref = P.Qap(inst.flow_matrix, inst.distance_matrix)
        elif kind == "jsp_int":
            ref = P.JspInt(inst.jobs)
        else:
            ref = P.Knapsack(inst.weights, inst.values, inst.capacity)
        custom = name in ("C2", "C2j")
        ops = G.tsp_delta_operators() if custom else ()
        oops = tuple((i, nm, f, 1.0) for i, nm, f in M.TSP_DELTA) if custom else ()
        out[name] = (prob, ref, ops, oops)
    return out
