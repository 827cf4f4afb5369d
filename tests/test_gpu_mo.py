"""Multi-objective routing on the device: objectives
("distance", "vehicles") (builtins.py:80-152), Weighted and Lexicographic
comparisons with tolerances (core.py:80-106, :315-347; engine.py:225-246), and
non-dominated-sort initialisation (engine.py:352-420).  The oracle reproduces
the reference on these runs bit-for-bit (tests/test_oracle_golden.py); here the
device run must be bit-identical to the oracle in Philox mode."""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2603_19163_b200 as G
from oracle import engine as OE
from oracle import problems as OP
from paper_2603_19163_b200 import instances as I
from paper_2603_19163_b200.core import Lexicographic, Weighted

pytestmark = pytest.mark.gpu

GOLD = json.loads((Path(__file__).with_name("golden") / "golden_mo.json").read_text())["runs"]


def _pair(g):
    inst, names, c = g["instance"], tuple(g["objectives_names"]), g["comparison"]
    kw, meta = {"objectives": names}, {"objectives": names}
    if c is not None and c[0] == "w":
        kw["weights"] = tuple(c[1])
        meta["comparison"] = Weighted(tuple(c[1]))
    elif c is not None:
        kw["lex"] = (tuple(c[1]), tuple(c[2]))
        meta["comparison"] = Lexicographic(tuple(c[1]), tuple(c[2]))
    if inst["tw"]:
        n, veh, seed = inst["vrptw_solomon_like"]
        vd = I.vrptw_solomon_like(n=n, vehicles=veh, seed=seed)
        prob = G.builtin_problem("vrptw", G.InstanceData(
            distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity,
            vehicles=vd.vehicles, ready_times=vd.ready, due_times=vd.due,
            service_times=vd.service, meta=meta))
        return prob, OP.Vrptw(vd.dist, vd.demands, vd.capacity, vd.vehicles, vd.ready, vd.due,
                              vd.service, **kw)
    d = np.array(inst["dist"])
    prob = G.builtin_problem("cvrp", G.InstanceData(
        distance_matrix=d, demands=np.array(inst["demands"]), capacity=inst["capacity"],
        vehicles=inst["vehicles"], meta=meta))
    return prob, OP.Routing(d, inst["demands"], inst["capacity"], inst["vehicles"], **kw)


@pytest.mark.parametrize("key", sorted(GOLD))
def test_multiobjective_run_bit_identical_to_oracle(key):
    g = GOLD[key]
    prob, ref = _pair(g)
    c = g["config"]
    kw = dict(population=c["population"], team_size=c["team_size"],
              max_generations=c["max_generations"], seed=c["seed"], record_history=True)
    res = G.run(prob, G.EngineConfig(islands=G.IslandsConfig(count=c["islands"],
                                                             migration="hybrid", interval=5),
                                     **kw))
    out = OE.run(ref, OE.RunCfg(islands=c["islands"], migration="hybrid", migration_interval=5,
                                allowed_ops=prob.device_sequences(), **kw),
                 device_stream="philox")
    assert res.device["error_flags"] == 0
    assert res.history["best_phi"] == out.history["best_phi"]
    assert res.objectives == out.objectives and res.penalty == out.penalty
    assert [e["weight"] for e in res.final_weights["sequences"]] == [float(w) for w in out.weights]
    got = [[[int(x) for x in s.row(r)] for r in range(s.d1)] for s in res.population]
    exp = [[[int(x) for x in s.row(r)] for r in range(s.d1)] for s in out.population]
    assert got == exp
    assert [list(s.objectives) for s in res.population] == [list(s.obj) for s in out.population]


def test_multiobjective_eval_vector():
    g = GOLD["vrptw30_lex"]
    prob, ref = _pair(g)
    import random
    sols = [OE.random_solution(ref.spec, random.Random(k)) for k in range(8)]
    obj, pen = G.problems.device_evaluate(prob, [G.Solution(s.data, s.sizes, 2) for s in sols])
    for s, o, p in zip(sols, obj, pen):
        OP.evaluate(ref, s)
        assert list(o) == list(s.obj) and p == s.pen
