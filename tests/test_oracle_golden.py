"""Pins the CPU oracle to the reference through the committed golden vectors
(tests/golden/make_golden.py).  CPU only."""

import math
import random

import numpy as np
import pytest

from oracle import aos as A
from oracle import engine as E
from oracle import moves as M
from oracle import problems as P
from oracle import rng as R
from tests.helpers import sol_from_json, sol_rows


def test_mix64_matches_reference(golden):
    for parts, h in golden["mix64"]:
        assert R.mix64(*parts) == h


def test_philox_known_answers():
    # Random123 kat_vectors, philox4x32 R=10
    assert R.philox4x32_10((0, 0, 0, 0), (0, 0)) == (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)
    assert R.philox4x32_10((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2) == \
        (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)
    assert R.philox4x32_10((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344),
                           (0xA4093822, 0x299F31D0)) == \
        (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)


def test_word_random_equals_cpython_random():
    for seed in (1, 99, R.mix64(42, 0, 1, 5, 0), 2 ** 64 - 3):
        a, b = random.Random(seed), R.WordRandom(R.mt_words(seed))
        for _ in range(500):
            assert a.random() == b.random()
            n = a.randrange(1, 700)
            assert n == b.randrange(1, 700)
            assert a.randrange(n) == b.randrange(n)
            assert a.randrange(1) == b.randrange(1)
            x, y = list(range(n % 50)), list(range(n % 50))
            a.shuffle(x)
            b.shuffle(y)
            assert x == y
            m = min(n, 40)
            assert a.sample(range(m), min(3, m)) == b.sample(range(m), min(3, m))
            assert a.sample(range(1, n + 2), 1) == b.sample(range(1, n + 2), 1)


def test_builtin_sum_is_neumaier():
    rng = random.Random(3)
    for _ in range(300):
        xs = [rng.uniform(-1, 1) * 10 ** rng.randrange(-8, 8) for _ in range(rng.randrange(1, 30))]
        assert sum(xs) == A.neumaier_sum(xs)
        assert float(sum(np.float64(x) for x in xs)) == math.fsum([]) + _seq(xs)


def _seq(xs):
    s = 0.0
    for x in xs:
        s += x
    return s


@pytest.mark.parametrize("name", ["tsp51", "tsp51f", "tsp442", "vrptw100", "qap100",
                                  "jsp20x15", "knap1000"])
def test_evaluate_matches_reference(golden, oracle_problems, name):
    p = oracle_problems[name]
    for row in golden["evaluate"][name]:
        s = sol_from_json(p, row)
        obj, pen = P.evaluate(p, s)
        assert [float(o) for o in obj] == row["obj"]
        assert pen == row["pen"]


def test_operators_match_reference(golden, oracle_problems):
    fns = {sid: fn for sid, _, fn in M.BUILTINS}
    fns.update({sid: fn for sid, _, fn in M.TSP_DELTA})
    for key, rows in golden["operators"].items():
        name, sid = key.split(":")
        p = oracle_problems[name]
        for row in rows:
            s = sol_from_json(p, row["before"])
            fns[int(sid)](s, R.WordRandom(R.mt_words(row["rng_seed"])), M.Ctx(p))
            assert sol_rows(s) == row["after"]["data"], key


def test_aos_updates_match_reference(golden):
    cfg = A.AosCfg()
    for row in golden["aos"]:
        caps = [math.inf if c is None else c for c in row["caps"]]
        reg = A.Registry([A.Entry(i, f"s{i}", None, w, 0.0, c)
                          for i, (w, c) in enumerate(zip(row["weights"], caps))])
        assert reg.weights() == row["normalized"]
        A.update_weights(reg, row["usage"], row["impr"], cfg)
        assert [float(w) for w in reg.weights()] == row["first"]
        usage2 = row["usage"][::-1]
        impr2 = [min(a, b) for a, b in zip(row["impr"][::-1], usage2)]
        A.update_weights(reg, usage2, impr2, cfg)
        assert [float(w) for w in reg.weights()] == row["second"]
        u3 = (row["usage"][:3] + [0, 0, 0])[:3]
        i3 = (row["impr"][:3] + [0, 0, 0])[:3]
        assert list(A.update_k(A.DEFAULT_K, u3, i3, cfg)) == row["k"]
        draws = [A.sample_seq(reg, R.WordRandom(R.mt_words(9000 + j))) for j in range(16)]
        assert draws == row["draws"]


def test_population_sizing_matches_reference(golden):
    for *args, expect in golden["sizing"]:
        assert E.population_size(*args) == expect


@pytest.mark.parametrize("key,name", [("tsp51", "tsp51"), ("tsp51_delta", "tsp51"),
                                      ("tsp51f", "tsp51f"), ("qap100", "qap100"),
                                      ("jsp20x15", "jsp20x15"), ("knap1000", "knap1000"),
                                      ("vrptw100", "vrptw100")])
def test_run_trajectory_matches_reference(golden, oracle_problems, key, name):
    g = golden["runs"][key]
    c = g["config"]
    isl = c["islands"]
    custom = tuple((sid, nm, fn, 1.0) for sid, nm, fn in M.TSP_DELTA) if c["custom"] else ()
    cfg = E.RunCfg(population=c["population"], team_size=c["team_size"],
                   max_generations=c["max_generations"], seed=c["seed"],
                   islands=isl["count"], migration=isl["migration"],
                   migration_interval=isl["interval"], top_n=isl["top_n"],
                   elite_interval=c.get("elite_injection_interval", 50),
                   custom_ops=custom, record_history=True)
    out = E.run(oracle_problems[name], cfg)
    assert sol_rows(out.best) == g["best"]["data"]
    assert out.objectives == g["objectives"] and out.penalty == g["penalty"]
    assert out.history["best_phi"] == g["history"]
    assert out.generations == g["generations"]
    assert out.ids == g["ids"]
    assert [float(w) for w in out.weights] == g["weights"]
    assert list(out.k_weights) == g["k_weights"]


def _mo_pair(g):
    """Oracle problem for a golden_mo.json run (and the product problem)."""
    inst, names, c = g["instance"], tuple(g["objectives_names"]), g["comparison"]
    kw = {"objectives": names}
    if c is not None and c[0] == "w":
        kw["weights"] = tuple(c[1])
    elif c is not None:
        kw["lex"] = (tuple(c[1]), tuple(c[2]))
    if inst["tw"]:
        from paper_2603_19163_b200 import instances as I
        n, veh, seed = inst["vrptw_solomon_like"]
        vd = I.vrptw_solomon_like(n=n, vehicles=veh, seed=seed)
        return P.Vrptw(vd.dist, vd.demands, vd.capacity, vd.vehicles, vd.ready, vd.due,
                        vd.service, **kw), vd
    return P.Routing(np.array(inst["dist"]), inst["demands"], inst["capacity"],
                      inst["vehicles"], **kw), inst


@pytest.mark.parametrize("key", ["cvrp8_w", "cvrp8_w100", "cvrp8_lex_veh", "cvrp8_lex_tol",
                                 "vrptw30_w", "vrptw30_lex"])
def test_multiobjective_run_matches_reference(key):
    """Bi-objective routing, Weighted and Lexicographic, non-dominated-sort init
    (engine.py:225-246, :352-420; core.py:315-347) — oracle in MT mode ==
    reference run() bit-for-bit."""
    import json
    from pathlib import Path
    g = json.loads((Path(__file__).with_name("golden") / "golden_mo.json").read_text())["runs"][key]
    prob, _ = _mo_pair(g)
    c = g["config"]
    out = E.run(prob, E.RunCfg(population=c["population"], team_size=c["team_size"],
                               max_generations=c["max_generations"], seed=c["seed"],
                               islands=c["islands"], migration="hybrid", migration_interval=5,
                               record_history=True))
    assert sol_rows(out.best) == g["best"]["data"]
    assert out.objectives == g["objectives"] and out.penalty == g["penalty"]
    assert out.history["best_phi"] == g["history"]
    assert [float(w) for w in out.weights] == g["weights"]
    assert list(out.k_weights) == g["k_weights"]


@pytest.mark.parametrize("key", ["assign40", "color40", "binpack30", "loadbal40", "vrpprio20",
                                 "vrpnl20", "jspperm6x4", "sched8x6"])
def test_extra_builtins_match_reference(key):
    """assignment / graph colouring / bin packing / load balancing / priority and
    nonlinear VRP (builtins.py:193-394): evaluations and a whole run == reference."""
    from tests.extra_problems import GOLD, oracle_problem, sol_rows as rows_of
    prob = oracle_problem(key)
    for row in GOLD["evaluate"][key]:
        s = P.Sol(*rows_of(row["data"], prob.spec.d2), 1)
        P.evaluate(prob, s)
        assert [float(s.obj[0])] == row["obj"] and s.pen == row["pen"]
    g = GOLD["runs"][key]
    c = g["config"]
    out = E.run(prob, E.RunCfg(population=c["population"], team_size=c["team_size"],
                               max_generations=c["max_generations"], seed=c["seed"],
                               record_history=True))
    assert sol_rows(out.best) == g["best"]["data"]
    assert out.objectives == g["objectives"] and out.penalty == g["penalty"]
    assert out.history["best_phi"] == g["history"]
    assert [float(w) for w in out.weights] == g["weights"]
