"""Exact optima and lower bounds for the BASELINE shapes (host, numpy) — the
references the gap@30 s figures are measured against (profiles/best_known.json):

* C5b knapsack n=1000: exact optimum by dynamic programming over capacity
* C2j jittered lattice: Held-Karp 1-tree lower bound (subgradient ascent)
* C5a JSP 20x15: max(longest job, busiest machine) lower bound
* C2: the lattice's known optimum 44,200 (even side: a unit-step Hamiltonian cycle)

    python tools/bounds.py            # prints JSON
"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2603_19163_b200 import instances as I  # noqa: E402


def knapsack_optimum(w, v, cap):
    w = np.asarray(w, dtype=np.int64)
    v = np.asarray(v, dtype=np.float64)
    cap = int(cap)
    best = np.zeros(cap + 1)
    for wi, vi in zip(w, v):
        if wi <= cap:
            cand = best[:cap + 1 - wi] + vi
            best[wi:] = np.maximum(best[wi:], cand)
    return float(best.max())


def _one_tree(c):
    """cost and node degrees of the minimum 1-tree (MST on 1..n-1 by Prim,
    plus node 0's two cheapest edges) for edge costs c."""
    n = len(c)
    sub = c[1:, 1:]
    m = n - 1
    in_tree = np.zeros(m, bool)
    in_tree[0] = True
    dist = sub[0].copy()
    parent = np.zeros(m, int)
    deg = np.zeros(n, int)
    cost = 0.0
    for _ in range(m - 1):
        j = int(np.argmin(np.where(in_tree, np.inf, dist)))
        cost += dist[j]
        deg[j + 1] += 1
        deg[parent[j] + 1] += 1
        in_tree[j] = True
        upd = (~in_tree) & (sub[j] < dist)
        dist[upd] = sub[j][upd]
        parent[upd] = j
    e = np.argsort(c[0, 1:])[:2] + 1
    cost += c[0, e[0]] + c[0, e[1]]
    deg[0] += 2
    deg[e] += 1
    return cost, deg


def one_tree_bound(d, upper, iters=4000):
    """Held-Karp bound: max over node penalties pi of the minimum 1-tree with
    edge costs d_ij + pi_i + pi_j, minus 2 sum(pi); Polyak steps toward the
    tour length `upper`, lambda halved after 50 iterations without progress."""
    d = np.asarray(d, dtype=np.float64)
    n = len(d)
    pi = np.zeros(n)
    best, lam, stall = -np.inf, 2.0, 0
    for _ in range(iters):
        cost, deg = _one_tree(d + pi[:, None] + pi[None, :])
        lb = cost - 2.0 * pi.sum()
        if lb > best + 1e-9:
            best, stall = lb, 0
        else:
            stall += 1
            if stall >= 50:
                lam, stall = lam / 2.0, 0
        g = (deg - 2).astype(np.float64)
        if not g.any() or lam < 1e-6:
            break
        pi += lam * (upper - lb) / float(g @ g) * g
    return float(best)


def vrptw_lateness_bound(inst):
    d, r, du = inst.distance_matrix, inst.ready_times, inst.due_times
    arr = np.maximum(r[1:], r[0] + d[0, 1:])
    return float(np.maximum(0.0, arr - du[1:]).sum())


def jsp_lower_bound(jobs):
    job = max(sum(t for _, t in ops) for ops in jobs)
    mach = {}
    for ops in jobs:
        for m, t in ops:
            mach[m] = mach.get(m, 0) + t
    return float(max(job, max(mach.values())))


def main():
    tab = I.baseline_instances()
    out = {}
    w, v, cap = tab["C5b"][1].weights, tab["C5b"][1].values, tab["C5b"][1].capacity
    out["C5b"] = {"optimum": knapsack_optimum(w, v, cap), "sense": "max",
                  "how": "exact dynamic programming over integer capacity"}
    out["C5a"] = {"lower_bound": jsp_lower_bound(tab["C5a"][1].jobs), "sense": "min",
                  "how": "max(longest job, busiest machine)"}
    out["C2"] = {"optimum": 44200.0, "sense": "min", "how": "unit-step Hamiltonian cycle"}
    out["C2j"] = {"lower_bound": one_tree_bound(tab["C2j"][1].distance_matrix, upper=45000.0),
                  "sense": "min",
                  "how": "Held-Karp 1-tree bound, subgradient ascent"}
    out["C3"] = {"penalty_lower_bound": vrptw_lateness_bound(tab["C3"][1]), "sense": "min",
                 "how": "sum over customers of max(0, max(ready, d(depot, c)) - due): lateness no "
                        "route can avoid (the R101 fixture is synthetic; 2 windows close before "
                        "the direct drive from the depot, so no zero-penalty solution exists)"}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
