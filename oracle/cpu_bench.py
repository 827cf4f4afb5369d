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
