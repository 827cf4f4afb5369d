"""The unmodified reference, timed on the host cores (bench.py's reference arm
and cpu_baseline legs).  Measurement infrastructure only: nothing in the
product imports it.

The reference package (pure Python + numpy) is installed by
tools/stage_reference.sh into baseline/_ref/ (git-ignored, shipped with the
repo snapshot).  Every measurement runs the reference's own public API —
`genopt.builtin_problem` + `genopt.run(problem, EngineConfig(...))` — in
independent processes, one per host core (its evolver threads are GIL-bound,
SURVEY §8d).  To time steady-state generations the only addition is a
timestamp at the first evolver of every generation (a wrapper around
genopt.engine.evolve_generation that calls the original unchanged).
When baseline/_ref is absent the oracle port (oracle/, pinned bit-for-bit to
the reference) stands in and the result says kind "port".
"""
from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
REF = ROOT / "baseline" / "_ref"


def available() -> bool:
    return (REF / "genopt" / "__init__.py").exists()


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _genopt():
    """Import the installed reference, never this repo's drop-in shim."""
    for k in [k for k in sys.modules if k == "genopt" or k.startswith("genopt.")]:
        del sys.modules[k]
    sys.path.insert(0, str(REF))  # ahead of the repo root and its genopt drop-in shim
    import genopt
    import genopt.demo_ops  # noqa: F401
    assert Path(genopt.__file__).resolve().is_relative_to(REF.resolve()), genopt.__file__
    return genopt


def _problem(g, workload):
    from paper_2603_19163_b200 import instances as I  # instance arrays only (numpy)
    kind, inst, _ = I.baseline_instances()[workload]
    fields = {k: v for k, v in vars(inst).items() if v is not None and k != "meta"}
    prob = g.builtin_problem(kind, g.InstanceData(**fields))
    ops = g.demo_ops.tsp_delta_operators() if workload in ("C2", "C2j") else ()
    return prob, ops


def _steady_worker(args):
    workload, seed, pop, team, warm, gens = args
    g = _genopt()
    prob, ops = _problem(g, workload)
    stamps = {}
    orig = g.engine.evolve_generation

    def timed(ev, ev_idx, generation, *a, **k):
        if ev_idx == 0 and generation not in stamps:
            stamps[generation] = time.perf_counter()
        return orig(ev, ev_idx, generation, *a, **k)

    g.engine.evolve_generation = timed
    cfg = g.EngineConfig(population=pop, team_size=team, max_generations=warm + gens, seed=seed,
                         custom_operators=ops)
    g.run(prob, cfg)
    t_end = time.perf_counter()
    return gens * pop * team, t_end - stamps[warm + 1]


def steady_throughput(workload: str, procs: int, pop: int = 8, team: int = 128, warm: int = 10,
                      gens: int = 4, seed: int = 42) -> dict:
    """Lane evaluations / s of generations warm+1 .. warm+gens, summed over
    `procs` concurrent processes (each its own seed)."""
    if not available():
        from oracle import cpu_bench
        return dict(cpu_bench.throughput_workload(workload, procs, pop, team, warm, gens, seed),
                    kind="port")
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_steady_worker, [(workload, seed + i, pop, team, warm, gens)
                                        for i in range(procs)])
    evals = sum(r[0] for r in res)
    wall = max(r[1] for r in res)
    return {"value": evals / wall, "evals": evals, "wall_s": wall, "procs": procs,
            "kind": "reference"}


def _gap_worker(args):
    workload, seed, seconds, best_known, sense = args
    g = _genopt()
    prob, ops = _problem(g, workload)
    cfg = g.EngineConfig(team_size=128, max_generations=10 ** 9, time_limit_seconds=seconds,
                         seed=seed, custom_operators=ops)
    r = g.run(prob, cfg)
    obj = float(r.objectives[0])
    return obj, r.penalty, r.generations_completed, r.config.get("population"), r.elapsed_seconds


def gap_at(workload: str, seconds: float, procs: int, best_known: float | None,
           sense: str = "min", seed: int = 1000) -> dict:
    """`procs` independent reference runs with a wall-clock budget (the
    reference's replicas semantics: the best counts, the median is reported
    beside it)."""
    if not available():
        from oracle import cpu_bench
        return dict(cpu_bench.gap_workload(workload, seconds, procs, best_known, sense, seed),
                    kind="port")
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_gap_worker, [(workload, seed + i, seconds, best_known, sense)
                                     for i in range(procs)])
    objs = sorted((r[0] for r in res if r[1] == 0.0), reverse=(sense == "max"))
    pens = sorted((float(r[1]), r[0]) for r in res)  # penalty first (core.py:315-347)
    out = {"best": objs[0] if objs else None, "median": objs[len(objs) // 2] if objs else None,
           "feasible_runs": len(objs), "procs": procs, "seconds": seconds,
           "best_penalty_objective": list(pens[0]),
           "median_penalty": pens[len(pens) // 2][0],
           "generations": sorted(r[2] for r in res), "kind": "reference"}
    if best_known and objs:
        sgn = 1.0 if sense == "min" else -1.0
        out["gap_pct"] = sgn * (objs[0] - best_known) / abs(best_known) * 100.0
        out["median_gap_pct"] = sgn * (out["median"] - best_known) / abs(best_known) * 100.0
    return out
