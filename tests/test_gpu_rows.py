"""GPU parity for the row kernel family (QAP / knapsack / JSP-int): device
evaluation against the oracle (bit-exact: all three BASELINE instances are
integer-valued) and whole evolve runs bit-identical to the oracle engine in
Philox mode with the same operator registry."""

import numpy as np
import pytest

import paper_2603_19163_b200 as G
from oracle import engine as OE
from oracle import problems as OP
from paper_2603_19163_b200 import instances as I
from tests.helpers import sol_from_json

pytestmark = pytest.mark.gpu


def _pair(name, small=False):
    if name == "qap":
        f, d = I.qap_random(30 if small else 100, 100)
        return (G.builtin_problem("qap", G.InstanceData(flow_matrix=f, distance_matrix=d)),
                OP.Qap(f, d))
    if name == "knap":
        w, v, cap = I.knapsack_random(200 if small else 1000, 1000)
        return (G.builtin_problem("knapsack", G.InstanceData(weights=w, values=v, capacity=cap)),
                OP.Knapsack(w, v, cap))
    jobs = I.jsp_random(6, 5, 7) if small else I.jsp_random(20, 15, 2015)
    return G.builtin_problem("jsp_int", G.InstanceData(jobs=jobs)), OP.JspInt(jobs)


@pytest.mark.parametrize("name,key", [("qap", "qap100"), ("knap", "knap1000"),
                                      ("jsp", "jsp20x15")])
def test_eval_matches_oracle_and_reference_golden(golden, name, key):
    prob, ref = _pair(name)
    sols = [sol_from_json(ref, row) for row in golden["evaluate"][key]]
    gsols = [G.Solution(s.data, s.sizes, 1) for s in sols]
    obj, pen = G.problems.device_evaluate(prob, gsols)
    for s, o, p, row in zip(sols, obj[:, 0], pen, golden["evaluate"][key]):
        assert [o] == row["obj"] and p == row["pen"]
    rng = np.random.default_rng(3)
    cfg = prob.config()
    extra = []
    for _ in range(32):
        s = OE.random_solution(ref.spec, __import__("random").Random(int(rng.integers(1e9))))
        extra.append(s)
    obj, pen = G.problems.device_evaluate(prob, [G.Solution(s.data, s.sizes, 1) for s in extra])
    for s, o, p in zip(extra, obj[:, 0], pen):
        OP.evaluate(ref, s)
        assert o == s.obj[0] and p == s.pen


@pytest.mark.parametrize("name,small,P,T,Gn,seed", [
    ("qap", True, 4, 32, 25, 11), ("qap", False, 2, 32, 6, 456),
    ("knap", True, 4, 32, 25, 12), ("knap", False, 2, 32, 8, 2024),
    ("jsp", True, 4, 16, 12, 13), ("jsp", False, 2, 16, 3, 789),
    # teams wider than the 384-thread row kernels: the 512-thread variants
    ("knap", True, 2, 448, 4, 31), ("jsp", True, 2, 448, 3, 32)])
def test_evolve_bit_identical_to_oracle(name, small, P, T, Gn, seed):
    prob, ref = _pair(name, small)
    res = G.run(prob, G.EngineConfig(population=P, team_size=T, max_generations=Gn, seed=seed,
                                     record_history=True))
    allowed = prob.device_sequences()
    out = OE.run(ref, OE.RunCfg(population=P, team_size=T, max_generations=Gn, seed=seed,
                                record_history=True, allowed_ops=allowed),
                 device_stream="philox")
    assert res.device["error_flags"] == 0
    assert res.generations_completed == out.generations
    assert [e["id"] for e in res.final_weights["sequences"]] == out.ids
    assert res.history["best_phi"] == out.history["best_phi"]
    assert res.objectives == out.objectives and res.penalty == out.penalty
    assert res.best.row(0).tolist() == out.best.row(0).tolist()
    assert [e["weight"] for e in res.final_weights["sequences"]] == [float(w) for w in out.weights]
    assert res.final_weights["k_steps"] == list(out.k_weights)
    assert [s.row(0).tolist() for s in res.population] == \
        [s.row(0).tolist() for s in out.population]


def test_knapsack_islands_and_migration():
    prob, ref = _pair("knap", True)
    kw = dict(population=6, team_size=32, max_generations=30, seed=5, record_history=True,
              elite_injection_interval=7)
    res = G.run(prob, G.EngineConfig(islands=G.IslandsConfig(count=3, migration="global_top_n",
                                                             interval=5, top_n=2), **kw))
    out = OE.run(ref, OE.RunCfg(islands=3, migration="global_top_n", migration_interval=5,
                                top_n=2, elite_interval=7, allowed_ops=prob.device_sequences(),
                                population=6, team_size=32, max_generations=30, seed=5,
                                record_history=True), device_stream="philox")
    assert res.history["best_phi"] == out.history["best_phi"]
    assert [s.row(0).tolist() for s in res.population] == \
        [s.row(0).tolist() for s in out.population]


def _vrptw_pair(n=None, vehicles=None, tw=True):
    vd = I.vrptw_solomon_like() if n is None else I.vrptw_solomon_like(n=n, vehicles=vehicles,
                                                                       seed=7)
    if tw:
        g = G.builtin_problem("vrptw", G.InstanceData(
            distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity,
            vehicles=vd.vehicles, ready_times=vd.ready, due_times=vd.due,
            service_times=vd.service))
        return g, OP.Vrptw(vd.dist, vd.demands, vd.capacity, vd.vehicles, vd.ready, vd.due,
                           vd.service)
    g = G.builtin_problem("cvrp", G.InstanceData(distance_matrix=vd.dist, demands=vd.demands,
                                                 capacity=vd.capacity, vehicles=vd.vehicles))
    return g, OP.Routing(vd.dist, vd.demands, vd.capacity, vd.vehicles)


def test_vrptw_eval_bit_exact_against_reference_golden(golden):
    prob, ref = _vrptw_pair()
    rows = golden["evaluate"]["vrptw100"]
    sols = [sol_from_json(ref, row) for row in rows]
    obj, pen = G.problems.device_evaluate(prob, [G.Solution(s.data, s.sizes, 1) for s in sols])
    for o, p, row in zip(obj[:, 0], pen, rows):
        assert [o] == row["obj"] and p == row["pen"]  # float64 bit-for-bit (numpy pairwise)


@pytest.mark.parametrize("tw,n,veh,P,T,Gn,seed", [(True, 30, 6, 4, 32, 20, 21),
                                                  (False, 30, 6, 4, 32, 20, 22),
                                                  (True, None, None, 2, 16, 4, 42),
                                                  (True, 30, 6, 2, 448, 3, 23)])
def test_routing_evolve_bit_identical_to_oracle(tw, n, veh, P, T, Gn, seed):
    prob, ref = _vrptw_pair(n, veh, tw)
    res = G.run(prob, G.EngineConfig(population=P, team_size=T, max_generations=Gn, seed=seed,
                                     record_history=True))
    out = OE.run(ref, OE.RunCfg(population=P, team_size=T, max_generations=Gn, seed=seed,
                                record_history=True, allowed_ops=prob.device_sequences()),
                 device_stream="philox")
    assert res.device["error_flags"] == 0
    assert res.history["best_phi"] == out.history["best_phi"]
    assert res.objectives == out.objectives and res.penalty == out.penalty
    assert [e["weight"] for e in res.final_weights["sequences"]] == [float(w) for w in out.weights]
    got = [([int(x) for x in s.row(r)] for r in range(s.d1)) for s in res.population]
    exp = [([int(x) for x in s.row(r)] for r in range(s.d1)) for s in out.population]
    assert [list(map(list, g)) for g in got] == [list(map(list, e)) for e in exp]


def test_qap_ox_crossover_uneven_islands():
    """OX mates come from the evolver's own island of the generation snapshot
    (engine.py:553-559, :687-689); 7 evolvers over 3 islands = sizes 3/2/2."""
    prob, ref = _pair("qap", True)
    kw = dict(population=7, team_size=32, max_generations=24, seed=77, record_history=True,
              elite_injection_interval=9)
    res = G.run(prob, G.EngineConfig(islands=G.IslandsConfig(count=3, migration="ring",
                                                             interval=8), **kw))
    out = OE.run(ref, OE.RunCfg(islands=3, migration="ring", migration_interval=8,
                                elite_interval=9, allowed_ops=prob.device_sequences(),
                                population=7, team_size=32, max_generations=24, seed=77,
                                record_history=True), device_stream="philox")
    assert 12 in [e["id"] for e in res.final_weights["sequences"]]
    assert res.history["best_phi"] == out.history["best_phi"]
    assert [e["weight"] for e in res.final_weights["sequences"]] == [float(w) for w in out.weights]
    assert [s.row(0).tolist() for s in res.population] == \
        [s.row(0).tolist() for s in out.population]


@pytest.mark.parametrize("name,extra,P,T,Gn,seed", [
    ("qap", 12, 3, 32, 6, 31), ("knap", 13, 3, 32, 6, 32), ("jsp", 13, 3, 16, 4, 33),
    ("vrptw", 12, 3, 16, 4, 34), ("cvrp", 12, 3, 16, 4, 35)])
def test_guided_rebuild_dominant_registry(name, extra, P, T, Gn, seed):
    """Registry restricted to guided_rebuild (+ the family's crossover), so most
    lanes run op_guided_rebuild (operators.py:501-571) with its phi-scored trials."""
    if name in ("vrptw", "cvrp"):
        prob, ref = _vrptw_pair(30, 6, name == "vrptw")
    else:
        prob, ref = _pair(name, True)
    ops = (16, extra)
    prob.device_sequences = lambda: ops
    res = G.run(prob, G.EngineConfig(population=P, team_size=T, max_generations=Gn, seed=seed,
                                     record_history=True))
    out = OE.run(ref, OE.RunCfg(population=P, team_size=T, max_generations=Gn, seed=seed,
                                record_history=True, allowed_ops=ops), device_stream="philox")
    assert res.device["error_flags"] == 0
    assert [e["id"] for e in res.final_weights["sequences"]] == out.ids
    assert res.history["best_phi"] == out.history["best_phi"]
    assert res.objectives == out.objectives and res.penalty == out.penalty
    got = [[[int(x) for x in s.row(r)] for r in range(s.d1)] for s in res.population]
    exp = [[[int(x) for x in s.row(r)] for r in range(s.d1)] for s in out.population]
    assert got == exp
