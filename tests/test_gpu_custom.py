"""NVRTC user problems (the paper's solve_custom; the
reference's ProblemDefinition callbacks, problems.py:49-74): objective and
penalty are CUDA snippets compiled into the row evolve kernel.  Each test
restates its snippet in Python for the oracle (same arithmetic order) and
requires device evaluation and whole runs to be bit-identical to the oracle
engine in Philox mode with the full registry of the encoding (crossovers and
guided rebuild included, whose trials call the snippet)."""

import random

import numpy as np
import pytest

import paper_2603_19163_b200 as G
from oracle import engine as OE
from oracle import problems as OP
from paper_2603_19163_b200 import _native as N
from paper_2603_19163_b200 import instances as I

pytestmark = pytest.mark.gpu

TOUR = """
  const int n = sol.n;
  double s = 0.0;
  for (int i = 0; i < n; ++i) {
    const int a = sol[i], b = sol[i + 1 == n ? 0 : i + 1];
    s += data.dist[a * n + b];
  }
  return s;
"""

KNAP_OBJ = """
  double v = 0.0;
  for (int i = 0; i < sol.n; ++i) v += data.value[i] * (double)sol[i];
  return v;
"""
KNAP_PEN = """
  double w = 0.0;
  for (int i = 0; i < sol.n; ++i) w += data.weight[i] * (double)sol[i];
  const double over = w - data.cap[0];
  return over > 0.0 ? over : 0.0;
"""

LOADS = """
  double load[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int i = 0; i < sol.n; ++i) load[sol[i]] += data.dur[i];
  double mx = 0.0;
  for (int m = 0; m < 8; ++m) mx = load[m] > mx ? load[m] : mx;
  return mx;
"""


def _tour_py(d):
    n = d.shape[0]

    def obj(t):
        s = 0.0
        for i in range(n):
            s += d[t[i], t[(i + 1) % n]]
        return s
    return obj


def _knap_py(w, v, cap):
    def obj(x):
        s = 0.0
        for i in range(len(x)):
            s += v[i] * float(x[i])
        return s

    def pen(x):
        s = 0.0
        for i in range(len(x)):
            s += w[i] * float(x[i])
        return max(0.0, s - cap) if s - cap > 0.0 else 0.0
    return obj, pen


def _loads_py(dur):
    def obj(x):
        load = [0.0] * 8
        for i in range(len(x)):
            load[int(x[i])] += dur[i]
        mx = 0.0
        for m in range(8):
            mx = load[m] if load[m] > mx else mx
        return mx
    return obj


def _cases():
    d = I.tsp_random(30, 7, True)
    rng = np.random.default_rng(11)
    w = rng.integers(1, 100, 60).astype(float)
    v = rng.integers(1, 100, 60).astype(float)
    cap = float(w.sum() // 2)
    dur = rng.integers(1, 50, 40).astype(float)
    ko, kp = _knap_py(w, v, cap)
    return {
        "tour": (G.CudaProblem("permutation", 30, TOUR, data={"dist": d}, init_matrices=[d]),
                 OP.Custom(OP.PERM, 30, _tour_py(d), mats=[d])),
        "knap": (G.CudaProblem("binary", 60, KNAP_OBJ, KNAP_PEN,
                               data={"value": v, "weight": w, "cap": [cap]}, maximize=True),
                 OP.Custom(OP.BINARY, 60, ko, kp, maximize=True)),
        "loads": (G.CudaProblem("integer", 40, LOADS, data={"dur": dur}, lb=0, ub=3),
                  OP.Custom(OP.INTEGER, 40, _loads_py(dur), lb=0, ub=3)),
    }


@pytest.mark.parametrize("name", ["tour", "knap", "loads"])
def test_user_objective_eval_matches_python(name):
    prob, ref = _cases()[name]
    r = random.Random(5)
    sols = [OE.random_solution(ref.spec, r) for _ in range(24)]
    obj, pen = G.problems.device_evaluate(prob, [G.Solution(s.data, s.sizes, 1) for s in sols])
    for s, o, p in zip(sols, obj[:, 0], pen):
        OP.evaluate(ref, s)
        assert o == s.obj[0] and p == s.pen


@pytest.mark.parametrize("name,P,T,Gn,seed", [("tour", 4, 32, 20, 3), ("knap", 4, 32, 20, 4),
                                              ("loads", 4, 32, 20, 5)])
def test_user_problem_run_bit_identical_to_oracle(name, P, T, Gn, seed):
    prob, ref = _cases()[name]
    res = G.run(prob, G.EngineConfig(population=P, team_size=T, max_generations=Gn, seed=seed,
                                     record_history=True))
    out = OE.run(ref, OE.RunCfg(population=P, team_size=T, max_generations=Gn, seed=seed,
                                record_history=True, allowed_ops=prob.device_sequences()),
                 device_stream="philox")
    assert res.device["error_flags"] == 0
    assert [e["id"] for e in res.final_weights["sequences"]] == out.ids
    assert res.history["best_phi"] == out.history["best_phi"]
    assert res.objectives == out.objectives and res.penalty == out.penalty
    assert [s.row(0).tolist() for s in res.population] == \
        [s.row(0).tolist() for s in out.population]


@pytest.mark.parametrize("name,ops", [("tour", (16, 12)), ("knap", (16, 13)), ("loads", (16, 13))])
def test_user_problem_guided_rebuild_dominant(name, ops):
    """guided_rebuild trials call the user objective on virtual rows."""
    prob, ref = _cases()[name]
    prob.device_sequences = lambda: ops
    res = G.run(prob, G.EngineConfig(population=3, team_size=16, max_generations=5, seed=9,
                                     record_history=True))
    out = OE.run(ref, OE.RunCfg(population=3, team_size=16, max_generations=5, seed=9,
                                record_history=True, allowed_ops=ops), device_stream="philox")
    assert res.history["best_phi"] == out.history["best_phi"]
    assert [[s.row(r).tolist() for r in range(s.d1)] for s in res.population] == \
        [[s.row(r).tolist() for r in range(s.d1)] for s in out.population]


def test_solve_custom_api_and_compile_errors():
    d = I.tsp_random(20, 3, True)
    res = G.solve_custom(encoding="permutation", dim2=20, n=20, compute_obj=TOUR,
                         data={"dist": d}, time_limit=1.0, seed=1)
    assert res.generations_completed > 0
    t = res.best.row(0)
    assert res.objectives[0] == sum(d[t[i], t[(i + 1) % 20]] for i in range(20))
    bad = G.CudaProblem("binary", 8, "return undefined_symbol;")
    with pytest.raises(N.NativeError) as e:
        bad.device_handle(0)
    assert e.value.status == N.GO_E_COMPILE and "undefined_symbol" in str(e.value)


@pytest.mark.parametrize("key", ["assign40", "color40", "binpack30", "loadbal40", "vrpprio20",
                                 "vrpnl20", "jspperm6x4", "sched8x6"])
def test_extra_builtins_on_device(key):
    """Further reference built-ins on the device (NVRTC objectives, partition
    variants): device evaluation equals the reference goldens; whole runs equal
    the oracle in Philox mode."""
    from tests.extra_problems import GOLD, oracle_problem, product_problem, sol_rows
    prob, ref = product_problem(key), oracle_problem(key)
    rows = GOLD["evaluate"][key]
    sols = [G.Solution(*sol_rows(r["data"], ref.spec.d2), 1) for r in rows]
    obj, pen = G.problems.device_evaluate(prob, sols)
    for o, p, r in zip(obj[:, 0], pen, rows):
        assert [o] == r["obj"] and p == r["pen"]
    res = G.run(prob, G.EngineConfig(population=4, team_size=32, max_generations=15, seed=3,
                                     record_history=True))
    out = OE.run(ref, OE.RunCfg(population=4, team_size=32, max_generations=15, seed=3,
                                record_history=True, allowed_ops=prob.device_sequences()),
                 device_stream="philox")
    assert res.history["best_phi"] == out.history["best_phi"]
    assert [[s.row(r).tolist() for r in range(s.d1)] for s in res.population] == \
        [[s.row(r).tolist() for r in range(s.d1)] for s in out.population]


@pytest.mark.parametrize("key,ops", [("jspperm6x4", (16, 12)), ("jspperm6x4", (14, 15, 4)),
                                     ("jspperm6x4", (0, 1, 2, 3)), ("sched8x6", (16, 13)),
                                     ("sched8x6", (6, 14, 15)), ("sched8x6", (5, 6, 13))])
def test_multi_fixed_rows_operator_mixes(key, ops):
    """MULTI_FIXED rows (jsp_perm permutation rows, schedule_binary cells):
    row draws (_pick_row / randrange(d1), operators.py:140-144, :450, :481,
    :519), per-row OX / shuffles / rebuilds with whole-solution trial scoring —
    bit-identical to the oracle with operator-dominated registries."""
    from tests.extra_problems import oracle_problem, product_problem
    prob, ref = product_problem(key), oracle_problem(key)
    prob.device_sequences = lambda: ops
    res = G.run(prob, G.EngineConfig(population=4, team_size=32, max_generations=12, seed=21,
                                     record_history=True))
    out = OE.run(ref, OE.RunCfg(population=4, team_size=32, max_generations=12, seed=21,
                                record_history=True, allowed_ops=ops), device_stream="philox")
    assert res.history["best_phi"] == out.history["best_phi"]
    assert [[s.row(r).tolist() for r in range(s.d1)] for s in res.population] == \
        [[s.row(r).tolist() for r in range(s.d1)] for s in out.population]


# ---- user operators on user problems (CustomOperator, operators.py:79-88, :634-669) --------
SWAP_KICK = """
  const int i = ctx.randbelow(ctx.n), j = ctx.randbelow(ctx.n);
  if (i != j) ctx.swap(i, j);
  if (ctx.random() < 0.3) {
    const int k = ctx.randrange(0, ctx.n);
    ctx.swap(k, k + 1 == ctx.n ? 0 : k + 1);
  }
"""
GREEDY_FLIP = """
  double best = 0.0;
  int bi = -1;
  for (int t = 0; t < 3; ++t) {  // best of three single flips, scored by ctx.phi()
    const int p = ctx.randbelow(ctx.n);
    ctx.set(p, 1 - ctx.get(p));
    const double f = ctx.phi();
    ctx.set(p, 1 - ctx.get(p));
    if (bi < 0 || f < best) { best = f; bi = p; }
  }
  ctx.set(bi, 1 - ctx.get(bi));
"""
BROKEN = "ctx.set(0, ctx.get(0) + ;"
OUT_OF_RANGE = "ctx.set(0, 7);"  # leaves the encoding: excluded by the probe


def _swap_kick_py(sol, rng, ctx):
    row = sol.data[0]
    n = len(row)
    i, j = rng.randrange(n), rng.randrange(n)
    if i != j:
        row[i], row[j] = row[j], row[i]
    if rng.random() < 0.3:
        k = rng.randrange(0, n)
        k2 = 0 if k + 1 == n else k + 1
        row[k], row[k2] = row[k2], row[k]


def _greedy_flip_py(sol, rng, ctx):
    row = sol.data[0]
    best, bi = 0.0, -1
    for _ in range(3):
        p = rng.randrange(len(row))
        row[p] = 1 - row[p]
        f = ctx.phi(sol)
        row[p] = 1 - row[p]
        if bi < 0 or f < best:
            best, bi = f, p
    row[bi] = 1 - row[bi]


@pytest.mark.parametrize("name,ops,P,T,Gn,seed", [
    ("tour", [(100, "swap_kick", SWAP_KICK, _swap_kick_py, 2.0)], 4, 32, 15, 5),
    ("knap", [(100, "greedy_flip", GREEDY_FLIP, _greedy_flip_py, 1.0),
              (101, "broken", BROKEN, None, 1.0), (102, "oob", OUT_OF_RANGE, None, 1.0)],
     4, 32, 15, 6)])
def test_user_operators_on_user_problems(name, ops, P, T, Gn, seed):
    """CUDA-snippet operators compete in AOS on a user problem; compile errors and
    invalid probe outputs exclude only that operator (operators.py:649-665); the
    run is bit-identical to the oracle with the Python restatements."""
    prob, ref = _cases()[name]
    cops = tuple(G.CustomOperator(i, nm, initial_weight=w, cuda=src) for i, nm, src, _, w in ops)
    with pytest.warns(RuntimeWarning) if len(ops) > 1 else _nullcontext():
        res = G.run(prob, G.EngineConfig(population=P, team_size=T, max_generations=Gn,
                                         seed=seed, record_history=True, custom_operators=cops))
    kept = [(i, nm, fn, w) for i, nm, _, fn, w in ops if fn is not None]
    assert [e["id"] for e in res.final_weights["sequences"]][-len(kept):] == [k[0] for k in kept]
    out = OE.run(ref, OE.RunCfg(population=P, team_size=T, max_generations=Gn, seed=seed,
                                record_history=True, allowed_ops=prob.device_sequences(),
                                custom_ops=tuple(kept)), device_stream="philox")
    assert res.history["best_phi"] == out.history["best_phi"]
    assert [e["weight"] for e in res.final_weights["sequences"]] == [float(w) for w in out.weights]
    assert [s.row(0).tolist() for s in res.population] == [s.row(0).tolist() for s in out.population]


class _nullcontext:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def test_solve_custom_with_user_operators():
    d = I.tsp_random(20, 3, True)
    r = G.solve_custom(encoding="permutation", dim2=20, compute_obj=TOUR, data={"dist": d},
                       custom_operators=[G.CustomOperator(100, "swap_kick", cuda=SWAP_KICK)],
                       time_limit=2.0, max_generations=200)
    assert any(e["id"] == 100 for e in r.final_weights["sequences"])
    assert r.feasible and sorted(r.best.row(0).tolist()) == list(range(20))


# ---- two-objective user problems (core.py:69-106, engine.py:225-246, :352-420) ------------
ASCENTS = """
  int k = 0;  // adjacent ascending pairs (to be maximised)
  for (int i = 0; i + 1 < sol.n; ++i) k += sol[i] < sol[i + 1];
  return (double)k;
"""


def _ascents_py(t):
    return float(sum(1 for i in range(len(t) - 1) if t[i] < t[i + 1]))


@pytest.mark.parametrize("mode", ["weighted", "lex"])
def test_two_objective_user_problem(mode):
    """(tour length Minimize, ascents Maximize) under Weighted((0.7, 0.3)) or
    Lexicographic((1, 0), (0, 2)): NSGA-II initial fronts, the Lexicographic
    delta with a Maximize objective, vector compare in the epilogue — equal to
    the oracle."""
    from paper_2603_19163_b200.core import Lexicographic, Weighted
    d = I.tsp_random(24, 17, True)
    if mode == "weighted":
        comp, kw = Weighted((0.7, 0.3)), dict(weights=(0.7, 0.3))
    else:
        comp, kw = Lexicographic((1, 0), (0.0, 2.0)), dict(lex=((1, 0), (0.0, 2.0)))
    prob = G.CudaProblem("permutation", 24, [TOUR, ASCENTS], data={"dist": d},
                         maximize=(False, True), name=("length", "ascents"), comparison=comp)
    ref = OP.Custom(OP.PERM, 24, [_tour_py(d), _ascents_py], maximize=(False, True), **kw)
    sols = [OE.random_solution(ref.spec, random.Random(s)) for s in range(6)]
    obj, _ = G.problems.device_evaluate(prob, [G.Solution(s.data, s.sizes, 2) for s in sols])
    for s, o in zip(sols, obj):
        OP.evaluate(ref, s)
        assert list(o) == list(s.obj)
    res = G.run(prob, G.EngineConfig(population=6, team_size=32, max_generations=20, seed=9,
                                     record_history=True))
    out = OE.run(ref, OE.RunCfg(population=6, team_size=32, max_generations=20, seed=9,
                                record_history=True, allowed_ops=prob.device_sequences()),
                 device_stream="philox")
    assert res.objectives == list(out.best.obj) and res.penalty == out.best.pen
    assert [s.row(0).tolist() for s in res.population] == [s.row(0).tolist() for s in out.population]
    assert [list(s.objectives) for s in res.population] == [list(s.obj) for s in out.population]
