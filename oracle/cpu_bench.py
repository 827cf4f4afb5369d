"""CPU baseline legs for bench.py (test/measurement infrastructure only).

Runs the oracle engine in MT mode — which reproduces the reference's
`genopt.run()` bit-for-bit (tests/test_oracle_golden.py) — with the
reference's full operator registry plus the tsp-delta user operators, as
independent processes on the host cores (threads are GIL-bound).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

from . import engine as E
from . import moves as M
from . import problems as P
from .rng import STREAM_INIT, mt_stream


def _throughput_worker(args):
    dist, seed, pop, team, gens = args
    prob = P.Tsp(dist)
    cfg = E.RunCfg(population=pop, team_size=team, max_generations=gens, seed=seed,
                   custom_ops=tuple((i, n, f, 1.0) for i, n, f in M.TSP_DELTA))
    t = time.perf_counter()
    out = E.run(prob, cfg)
    wall = time.perf_counter() - t
    return out.lane_evals, wall, out.generations


def throughput(dist, procs: int, pop: int = 8, team: int = 128, gens: int = 4, seed: int = 42):
    """Aggregate lane evaluations / s over `procs` concurrent processes."""
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        t = time.perf_counter()
        res = pool.map(_throughput_worker, [(dist, seed + i, pop, team, gens)
                                            for i in range(procs)])
        wall = time.perf_counter() - t
    evals = sum(r[0] for r in res)
    return {"evals": evals, "wall_s": wall, "value": evals / wall, "procs": procs,
            "per_proc": [r[0] / r[1] for r in res]}


def _gap_worker(args):
    dist, seed, seconds, best_known = args
    prob = P.Tsp(dist)
    cfg = E.RunCfg(population=None, team_size=128, max_generations=10 ** 9,
                   time_limit_seconds=seconds, seed=seed, concurrency_hint=os.cpu_count() or 1,
                   custom_ops=tuple((i, n, f, 1.0) for i, n, f in M.TSP_DELTA))
    out = E.run(prob, cfg, best_known=best_known)
    return out.objectives[0], out.gap_pct, out.lane_evals, out.elapsed, out.generations


def gap_at(dist, seconds: float, procs: int, best_known: float, seed: int = 42):
    """Each process runs the reference pipeline with a wall-clock budget;
    best-of-N is the reference's `replicas` semantics (engine.py:605-614)."""
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        res = pool.map(_gap_worker, [(dist, seed + i, seconds, best_known) for i in range(procs)])
    gaps = sorted(r[1] for r in res)
    evals = sum(r[2] for r in res)
    wall = max(r[3] for r in res)
    return {"best_gap_pct": gaps[0], "median_gap_pct": gaps[len(gaps) // 2],
            "evals_per_s": evals / wall, "generations": [r[4] for r in res], "procs": procs}


def workload_problem(name):
    """An oracle problem for a BASELINE workload (instances.baseline_instances)."""
    from paper_2603_19163_b200 import instances as I
    kind, inst, _ = I.baseline_instances()[name]
    if kind == "tsp":
        return P.Tsp(inst.distance_matrix)
    if kind == "vrptw":
        return P.Vrptw(inst.distance_matrix, inst.demands, inst.capacity, inst.vehicles,
                       inst.ready_times, inst.due_times, inst.service_times)
    if kind == "qap":
        return P.Qap(inst.flow_matrix, inst.distance_matrix)
    if kind == "jsp_int":
        return P.JspInt(inst.jobs)
    return P.Knapsack(inst.weights, inst.values, inst.capacity)


def _ops(name):
    return tuple((i, n, f, 1.0) for i, n, f in M.TSP_DELTA) if name in ("C2", "C2j") else ()


def _steady_worker(args):
    name, seed, pop, team, warm, gens = args
    prob = workload_problem(name)
    t = time.perf_counter()
    E.run(prob, E.RunCfg(population=pop, team_size=team, max_generations=warm, seed=seed,
                         custom_ops=_ops(name)))
    t_warm = time.perf_counter() - t
    t = time.perf_counter()
    out = E.run(prob, E.RunCfg(population=pop, team_size=team, max_generations=warm + gens,
                               seed=seed, custom_ops=_ops(name)))
    return gens * pop * team, max(1e-9, time.perf_counter() - t - t_warm), out.generations


def throughput_workload(name, procs, pop=8, team=128, warm=2, gens=2, seed=42):
    """Port stand-in for baseline.refbench.steady_throughput: the warm-up is
    timed separately and subtracted (runs are deterministic)."""
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_steady_worker, [(name, seed + i, pop, team, warm, gens)
                                        for i in range(procs)])
    evals = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return {"value": evals / wall, "evals": evals, "wall_s": wall, "procs": procs}


def _gap_worker2(args):
    name, seed, seconds = args
    out = E.run(workload_problem(name), E.RunCfg(population=None, team_size=128,
                                                 max_generations=10 ** 9,
                                                 time_limit_seconds=seconds, seed=seed,
                                                 concurrency_hint=os.cpu_count() or 1,
                                                 custom_ops=_ops(name)))
    return out.objectives[0], out.penalty, out.generations


def gap_workload(name, seconds, procs, best_known, sense="min", seed=1000):
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_gap_worker2, [(name, seed + i, seconds) for i in range(procs)])
    objs = sorted((r[0] for r in res if r[1] == 0.0), reverse=(sense == "max"))
    out = {"best": objs[0] if objs else None, "median": objs[len(objs) // 2] if objs else None,
           "feasible_runs": len(objs), "procs": procs, "seconds": seconds,
           "generations": sorted(r[2] for r in res)}
    if best_known and objs:
        sgn = 1.0 if sense == "min" else -1.0
        out["gap_pct"] = sgn * (objs[0] - best_known) / abs(best_known) * 100.0
        out["median_gap_pct"] = sgn * (out["median"] - best_known) / abs(best_known) * 100.0
    return out
