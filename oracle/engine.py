"""Evolution loop restatement (test infrastructure only).

Restates `engine.py`: solution construction (:252-324), oversampled
initialisation (:327-360), cache-aware sizing (:426-461), island migration and
elite injection (:467-532), `evolve_generation` (:538-595) and the run loop
(:601-811).  `run(..., device_stream=...)` selects the word generator behind
the streams the GPU owns (lane :568, accept :587, migration :738):

    device_stream="mt"      -> the reference, bit-for-bit
    device_stream="philox"  -> the GPU engine, bit-for-bit (integer instances)

Host-side streams (init :647, probe :626) are MT19937 in both modes because
the product initialises the population on the host exactly like the reference.
"""

from __future__ import annotations

import math
import time
import warnings
from dataclasses import dataclass, field
from functools import cmp_to_key

import numpy as np

from . import aos as A
from . import moves as M
from .problems import (MAX, MIN, MULTI_FIXED, PARTITION, PERM, SINGLE, BINARY,
                       Sol, acceptance_delta, compare, evaluate, scalar_fitness,
                       validate)
from .rng import (STREAM_ACCEPT, STREAM_INIT, STREAM_LANE, STREAM_MIGRATION,
                  STREAM_PROBE, STREAMS, mt_stream, philox_stream)


# -- construction -------------------------------------------------------------

def random_solution(spec, rng) -> Sol:
    """engine.py:252-287."""
    data = np.zeros((spec.d1, spec.d2), dtype=np.int64)
    sizes = np.zeros(spec.d1, dtype=np.int64)
    if spec.kind == PERM:
        if spec.row_mode in (SINGLE, MULTI_FIXED):
            for r in range(1 if spec.row_mode == SINGLE else spec.d1):
                perm = list(range(spec.n))
                rng.shuffle(perm)
                data[r, :spec.n] = perm
                sizes[r] = spec.n
        else:
            vals = list(range(spec.n))
            rng.shuffle(vals)
            for v in vals:
                open_rows = [r for r in range(spec.d1) if sizes[r] < spec.d2]
                r = open_rows[rng.randrange(len(open_rows))]
                data[r, sizes[r]] = v
                sizes[r] += 1
    else:
        lo, hi = (0, 1) if spec.kind == BINARY else (spec.lb, spec.ub)
        for r in range(spec.d1):
            sizes[r] = spec.d2
            for p in range(spec.d2):
                data[r, p] = rng.randrange(lo, hi + 1)
    return Sol(data, sizes, spec.m)


def heuristic_perms(matrix):
    """engine.py:290-301."""
    m = np.asarray(matrix, dtype=np.float64)
    ra = np.argsort(m.sum(axis=1), kind="stable")
    ca = np.argsort(m.sum(axis=0), kind="stable")
    return [ra.astype(np.int64), ra[::-1].astype(np.int64),
            ca.astype(np.int64), ca[::-1].astype(np.int64)]


def perm_to_sol(perm, spec) -> Sol:
    """engine.py:304-324."""
    data = np.zeros((spec.d1, spec.d2), dtype=np.int64)
    sizes = np.zeros(spec.d1, dtype=np.int64)
    if spec.row_mode == SINGLE:
        data[0, :spec.n] = perm
        sizes[0] = spec.n
    elif spec.row_mode == MULTI_FIXED:
        for r in range(spec.d1):
            data[r, :spec.n] = perm
            sizes[r] = spec.n
    else:
        base, extra = divmod(spec.n, spec.d1)
        at = 0
        for r in range(spec.d1):
            size = base + (1 if r < extra else 0)
            data[r, :size] = perm[at:at + size]
            sizes[r] = size
            at += size
    return Sol(data, sizes, spec.m)


def init_population(problem, pop_size, oversample, rng):
    """engine.py:327-360 (single-objective branch)."""
    spec = problem.spec
    return _init_from_pool(problem, pop_size,
                           [random_solution(spec, rng) for _ in range(oversample * pop_size)])


def init_population_philox(problem, pop_size, oversample, seed, salt=0):
    """The GPU engine's device-side initialisation (EngineConfig.device_init,
    csrc/kernels/go_init.cuh): random solution i is drawn, in the reference's
    draw order (engine.py:252-287), from its own stream
    philox_stream(seed, STREAM_INIT, salt, i); the heuristic candidates and the
    selection are engine.py:327-360's."""
    spec = problem.spec
    pool = [random_solution(spec, philox_stream(seed, STREAM_INIT, salt, i))
            for i in range(oversample * pop_size)]
    return _init_from_pool(problem, pop_size, pool)


def _init_from_pool(problem, pop_size, pool):
    spec = problem.spec
    if spec.kind == PERM:
        for mat in problem.matrices():
            if mat.shape == (spec.n, spec.n):
                pool.extend(perm_to_sol(p, spec) for p in heuristic_perms(mat))
    for s in pool:
        evaluate(problem, s)
    if spec.m != 1:  # engine.py:352-360: non-dominated fronts, crowding order
        fronts = nondominated_sort(np.array([s.obj for s in pool]), spec.directions)
        keep = []
        for front in fronts:
            for idx in front:
                if len(keep) < pop_size:
                    keep.append(pool[idx])
        return keep
    pool.sort(key=cmp_to_key(lambda a, b: compare(problem, a, b)))
    return pool[:pop_size]


def nondominated_sort(points, directions):
    """engine.py:370-420 (fast_nondominated_sort + crowding order)."""
    pts = np.asarray(points, dtype=np.float64).copy()
    for j, d in enumerate(directions):
        if d == MAX:
            pts[:, j] = -pts[:, j]
    n = len(pts)

    def dom(a, b):
        return bool(np.all(a <= b) and np.any(a < b))
    dominated_by = [[] for _ in range(n)]
    count = np.zeros(n, dtype=np.int64)
    fronts = [[]]
    for i in range(n):
        for j in range(i + 1, n):
            if dom(pts[i], pts[j]):
                dominated_by[i].append(j)
                count[j] += 1
            elif dom(pts[j], pts[i]):
                dominated_by[j].append(i)
                count[i] += 1
    for i in range(n):
        if count[i] == 0:
            fronts[0].append(i)
    f = 0
    while fronts[f]:
        nxt = []
        for p in fronts[f]:
            for q in dominated_by[p]:
                count[q] -= 1
                if count[q] == 0:
                    nxt.append(q)
        f += 1
        fronts.append(nxt)
    fronts.pop()
    out = []
    for front in fronts:
        if len(front) <= 2:
            out.append(list(front))
            continue
        crowd = np.zeros(len(front))
        sub = pts[front]
        for j in range(sub.shape[1]):
            order = np.argsort(sub[:, j], kind="stable")
            span = sub[order[-1], j] - sub[order[0], j]
            crowd[order[0]] = crowd[order[-1]] = math.inf
            if span == 0:
                continue
            for pos in range(1, len(front) - 1):
                crowd[order[pos]] += (sub[order[pos + 1], j] - sub[order[pos - 1], j]) / span
        ranked = sorted(range(len(front)), key=lambda i: (-crowd[i], i))
        out.append([front[i] for i in ranked])
    return out


# -- sizing (engine.py:426-461) -----------------------------------------------

def pow2_ceil(x):
    p = 1
    while p < x:
        p <<= 1
    return p


def pow2_floor(x):
    p = 1
    while p * 2 <= x:
        p <<= 1
    return p


def population_size(hint, cache_budget, working_set, fast_budget):
    if min(hint, cache_budget, working_set, fast_budget) <= 0:
        raise ValueError("all sizing inputs must be positive")
    p_sm = max(2, pow2_ceil(hint))
    if working_set <= fast_budget:
        return p_sm
    ratio = cache_budget / working_set
    if ratio >= p_sm / 2:
        return p_sm
    return max(2, pow2_floor(ratio))


# -- population management (engine.py:467-532) --------------------------------

def best_index(problem, pop):
    b = 0
    for i in range(1, len(pop)):
        if compare(problem, pop[i], pop[b]) == -1:
            b = i
    return b


def worst_index(problem, pop):
    w = 0
    for i in range(1, len(pop)):
        if compare(problem, pop[i], pop[w]) == 1:
            w = i
    return w


def migrate(problem, pops, strategy, rng, top_n=1):
    k = len(pops)
    if k < 2:
        return
    if strategy == "ring":
        donors = [p[best_index(problem, p)].clone() for p in pops]
        for i in range(k):
            recv = pops[(i + 1) % k]
            if len(recv) == 1:
                if compare(problem, donors[i], recv[0]) == -1:
                    recv[0] = donors[i]
                continue
            w, b = worst_index(problem, recv), best_index(problem, recv)
            if w != b:
                recv[w] = donors[i]
        return
    flat = [s for p in pops for s in p]
    order = sorted(range(len(flat)), key=cmp_to_key(lambda a, b: compare(problem, flat[a], flat[b])))
    donors = [flat[i].clone() for i in order[:top_n]]
    for p in pops:
        b = best_index(problem, p)
        slots = [i for i in range(len(p)) if i != b]
        for d in donors:
            if not slots:
                break
            p[slots[rng.randrange(len(slots))]] = d.clone()


def island_members(pop_size, count):
    """engine.py:790-798."""
    base, extra = divmod(pop_size, count)
    out, at = [], 0
    for i in range(count):
        size = base + (1 if i < extra else 0)
        out.append(list(range(at, at + size)))
        at += size
    return out


# -- one generation (engine.py:538-595) ---------------------------------------

@dataclass
class Evolver:
    cur: Sol
    island: int
    usage: np.ndarray
    impr: np.ndarray
    k_usage: np.ndarray = field(default_factory=lambda: np.zeros(3, np.int64))
    k_impr: np.ndarray = field(default_factory=lambda: np.zeros(3, np.int64))


def evolve_generation(problem, ev, ev_idx, gen, temp, reg, kw, seed, team, pw,
                      snapshot, member_pos, stream, trace=None):
    cur = ev.cur

    def phi(s):
        evaluate(problem, s)
        return scalar_fitness(problem, s, pw)

    def pick_mate(rng):
        if len(snapshot) <= 1:
            return None
        j = rng.randrange(len(snapshot) - 1)
        return snapshot[j + (j >= member_pos)]

    ctx = M.Ctx(problem, pick_mate=pick_mate, phi=phi)
    fns = {e.id: e.fn for e in reg.entries}
    best_d, best, best_seqs, best_k = math.inf, None, [], 1
    for lane in range(team):
        rng = stream(seed, ev_idx, gen, lane, STREAM_LANE)
        k = A.sample_k(kw, rng)
        cand = cur.clone()
        seqs = []
        for _ in range(k):
            sid = A.sample_seq(reg, rng)
            seqs.append(sid)
            fns[sid](cand, rng, ctx)
        evaluate(problem, cand)
        d = acceptance_delta(problem, cand, cur, pw)
        if trace is not None:
            trace.append((ev_idx, gen, lane, k, tuple(seqs), d))
        if d < best_d:
            best_d, best, best_seqs, best_k = d, cand, seqs, k
    accept = best_d < 0
    if not accept and best is not None and temp > 0:
        accept = stream(seed, ev_idx, gen, 0, STREAM_ACCEPT).random() < math.exp(-best_d / temp)
    if accept and best is not None:
        improved = best_d < 0
        ev.cur = best
        pos = {sid: i for i, sid in enumerate(reg.ids())}
        for sid in best_seqs:
            ev.usage[pos[sid]] += 1
            ev.impr[pos[sid]] += improved
        ev.k_usage[best_k - 1] += 1
        ev.k_impr[best_k - 1] += improved
    return accept


# -- run loop (engine.py:601-811) ---------------------------------------------

@dataclass
class RunCfg:
    """The EngineConfig fields the loop reads (engine.py:108-129)."""

    population: int | None = None
    team_size: int = 128
    max_generations: int = 1000
    time_limit_seconds: float | None = None
    seed: int = 42
    initial_temperature: float | None = None
    cooling_alpha: float = 0.999
    oversample_factor: int = 4
    islands: int = 1
    migration: str = "ring"
    migration_interval: int = 100
    top_n: int = 1
    elite_interval: int = 50
    replicas: int = 1
    cache_budget_bytes: int = 32 * 1024 * 1024
    concurrency_hint: int = 8
    fast_budget_bytes: int = 96 * 1024
    working_set_bytes: int | None = None
    aos: A.AosCfg = field(default_factory=A.AosCfg)
    custom_ops: tuple = ()          # (id, name, fn, initial_weight)
    target_objective: float | None = None
    record_history: bool = False
    allowed_ops: tuple | None = None  # restrict build_registry
    device_init: bool = False       # the GPU engine's Philox initialisation (init_population_philox)


@dataclass
class RunOut:
    best: Sol
    objectives: list
    penalty: float
    feasible: bool
    gap_pct: float | None
    generations: int
    elapsed: float
    weights: list
    ids: list
    k_weights: tuple
    population: list
    history: dict | None
    lane_evals: int
    penalty_weight: float
    t0: float


def run(problem, cfg: RunCfg, best_known=None, device_stream="mt", trace=None,
        initial_population=None, workers=1):
    """`workers` > 1 evolves the evolvers of each generation in that many forked
    processes (evolvers are independent within a generation given the island
    snapshot, engine.py:687-701), so the oracle can check the device at the
    benchmark's own population sizes; results are identical to workers=1."""
    if cfg.replicas == 1:
        return run_single(problem, cfg, cfg.seed, best_known, device_stream, trace,
                          initial_population, workers)
    outs = [run_single(problem, cfg, cfg.seed + i, best_known, device_stream)
            for i in range(cfg.replicas)]
    best = outs[0]
    for o in outs[1:]:
        if compare(problem, o.best, best.best) == -1:
            best = o
    return best


def working_set(problem):
    """engine.py:459-461."""
    return problem.payload_nbytes() + problem.spec.d1 * problem.spec.d2 * 4


_PAR = {}


def _evolve_chunk(idxs):
    """Worker body of run_single(workers > 1): the generation's context is
    inherited through fork (_PAR)."""
    c = _PAR
    out = []
    for e_idx in idxs:
        ev = c["evs"][e_idx]
        evolve_generation(c["problem"], ev, e_idx, c["gen"], c["temp"], c["reg"], c["kw"],
                          c["seed"], c["team"], c["pw"], c["snaps"][ev.island],
                          c["member_pos"][e_idx], c["stream"])
        out.append((e_idx, ev))
    return out


def run_single(problem, cfg: RunCfg, seed, best_known=None, device_stream="mt",
               trace=None, initial_population=None, workers=1):
    t_start = time.perf_counter()
    stream = STREAMS[device_stream]
    spec = problem.spec
    reg = A.build_registry(spec, cfg.allowed_ops)
    A.apply_preset(reg, A.scale_of(spec))
    if cfg.custom_ops:
        probe_sol = random_solution(spec, mt_stream(seed, STREAM_PROBE))
        evaluate(problem, probe_sol)
        probe_ctx = M.Ctx(problem, pick_mate=lambda r: None,
                          phi=lambda s: (evaluate(problem, s), scalar_fitness(problem, s, 1.0))[1])
        for sid, name, fn, w in cfg.custom_ops:
            if sid < 100 or sid in reg.ids():
                raise ValueError(f"bad custom operator id {sid}")
            trial = probe_sol.clone()
            try:
                fn(trial, mt_stream(seed, STREAM_PROBE, sid), probe_ctx)
                ok = validate(problem, trial)
            except Exception as exc:  # noqa: BLE001 — mirrors operators.py:649-657
                warnings.warn(f"custom operator {name!r} excluded: {exc!r}", RuntimeWarning)
                continue
            if not ok:
                warnings.warn(f"custom operator {name!r} excluded: invalid probe output",
                              RuntimeWarning)
                continue
            A.add_custom(reg, sid, name, fn, w)

    if cfg.population is not None:
        pop_size = cfg.population
    else:
        pop_size = population_size(cfg.concurrency_hint, cfg.cache_budget_bytes,
                                   cfg.working_set_bytes or working_set(problem),
                                   cfg.fast_budget_bytes)
    pop_size = max(pop_size, cfg.islands)
    if initial_population is None and cfg.device_init:
        pop = init_population_philox(problem, pop_size, cfg.oversample_factor, seed)
    elif initial_population is None:
        pop = init_population(problem, pop_size, cfg.oversample_factor,
                              mt_stream(seed, STREAM_INIT))
    else:
        pop = [s.clone() for s in initial_population]
        for s in pop:
            evaluate(problem, s)

    if spec.penalty_weight is not None:
        pw = spec.penalty_weight
    else:
        scale = float(np.mean([abs(s.obj[0]) for s in pop]))
        pw = 1000.0 * (scale if scale > 0 else 1.0)

    isl = island_members(pop_size, cfg.islands)
    nseq = len(reg.entries)
    evs = [Evolver(pop[i], iid, np.zeros(nseq, np.int64), np.zeros(nseq, np.int64))
           for iid, members in enumerate(isl) for i in members]
    member_pos = [p for members in isl for p in range(len(members))]

    gbest = pop[best_index(problem, pop)].clone()
    t0 = cfg.initial_temperature
    if t0 is None:
        t0 = max(1e-6, 0.05 * abs(scalar_fitness(problem, gbest, pw)))
    kw = A.DEFAULT_K
    stall = 0
    mig_events = 0
    hist = {"best_phi": [], "temperature": []} if cfg.record_history else None
    done = 0
    lane_evals = 0
    for gen in range(1, cfg.max_generations + 1):
        if cfg.time_limit_seconds is not None and \
                time.perf_counter() - t_start >= cfg.time_limit_seconds:
            break
        temp = t0 * cfg.cooling_alpha ** (gen - 1)
        snaps = [[evs[i].cur for i in members] for members in isl]
        if workers > 1 and trace is None:
            import multiprocessing as mp
            _PAR.update(problem=problem, evs=evs, gen=gen, temp=temp, reg=reg, kw=kw, seed=seed,
                        team=cfg.team_size, pw=pw, snaps=snaps, member_pos=member_pos,
                        stream=stream)
            with mp.get_context("fork").Pool(workers) as pool:
                parts = pool.map(_evolve_chunk, [list(range(w, len(evs), workers))
                                                 for w in range(workers)])
            _PAR.clear()
            for part in parts:
                for e_idx, ev in part:
                    evs[e_idx] = ev
        else:
            for e_idx, ev in enumerate(evs):
                evolve_generation(problem, ev, e_idx, gen, temp, reg, kw, seed, cfg.team_size,
                                  pw, snaps[ev.island], member_pos[e_idx], stream, trace)
        lane_evals += len(evs) * cfg.team_size
        improved = False
        for ev in evs:
            if compare(problem, ev.cur, gbest) == -1:
                gbest = ev.cur.clone()
                improved = True
        stall = 0 if improved else stall + 1
        done = gen
        if hist is not None:
            hist["best_phi"].append(scalar_fitness(problem, gbest, pw))
            hist["temperature"].append(temp)
        if _target(problem, gbest, cfg.target_objective):
            break
        if gen % cfg.aos.interval == 0:
            usage = sum(ev.usage for ev in evs)
            impr = sum(ev.impr for ev in evs)
            ku = sum(ev.k_usage for ev in evs)
            ki = sum(ev.k_impr for ev in evs)
            for ev in evs:
                ev.usage[:] = 0
                ev.impr[:] = 0
                ev.k_usage[:] = 0
                ev.k_impr[:] = 0
            A.update_weights(reg, usage, impr, cfg.aos)
            kw = A.update_k(kw, ku, ki, cfg.aos)
            kw, stall = A.stagnation(stall, kw, cfg.aos)
        if cfg.islands >= 2 and gen % cfg.migration_interval == 0:
            strat = cfg.migration
            if strat == "hybrid":
                strat = "ring" if mig_events % 2 == 0 else "global_top_n"
            pops = [[evs[i].cur for i in members] for members in isl]
            migrate(problem, pops, strat, stream(seed, STREAM_MIGRATION, mig_events), cfg.top_n)
            for members, p in zip(isl, pops):
                for i, s in zip(members, p):
                    evs[i].cur = s
            mig_events += 1
        if gen % cfg.elite_interval == 0:
            cur = [ev.cur for ev in evs]
            evs[worst_index(problem, cur)].cur = gbest.clone()

    elapsed = time.perf_counter() - t_start
    gap = None
    if best_known is not None and spec.m == 1 and spec.directions[0] == MIN and best_known != 0:
        gap = (float(gbest.obj[0]) - best_known) / best_known * 100.0
    return RunOut(best=gbest, objectives=[float(v) for v in gbest.obj], penalty=float(gbest.pen),
                  feasible=gbest.pen == 0.0, gap_pct=gap, generations=done, elapsed=elapsed,
                  weights=reg.weights(), ids=reg.ids(), k_weights=tuple(kw),
                  population=[ev.cur for ev in evs], history=hist, lane_evals=lane_evals,
                  penalty_weight=pw, t0=t0)


def _target(problem, best, target):
    """engine.py:805-811."""
    if target is None or problem.spec.m != 1 or best.pen > 0:
        return False
    v = float(best.obj[0])
    if problem.spec.directions[0] == MIN:
        return v <= target + 1e-9
    return v >= target - 1e-9
