"""Launch-shape sweep: team sizes that are not multiples of 32 (padding lanes),
single-team and partial CTAs, one-evolver populations and the 512-lane maximum,
for each kernel family — bit-identical to the oracle (engine.py:563-595
semantics do not depend on how lanes map to warps)."""

import numpy as np
import pytest

import paper_2603_19163_b200 as G
from oracle import engine as OE
from oracle import moves as OM
from oracle import problems as OP
from paper_2603_19163_b200 import instances as I

pytestmark = pytest.mark.gpu

SHAPES = [(8, 1), (20, 3), (33, 7), (96, 2), (256, 3), (512, 1)]


def _pair(kind):
    if kind == "tsp":
        d = I.tsp_random(40, 3)
        return G.builtin_problem("tsp", G.InstanceData(distance_matrix=d)), OP.Tsp(d), True
    if kind == "knap":
        w, v, cap = I.knapsack_random(80, 5)
        return (G.builtin_problem("knapsack", G.InstanceData(weights=w, values=v, capacity=cap)),
                OP.Knapsack(w, v, cap), False)
    vd = I.vrptw_solomon_like(n=15, vehicles=4, seed=9)
    return (G.builtin_problem("cvrp", G.InstanceData(distance_matrix=vd.dist, demands=vd.demands,
                                                     capacity=vd.capacity, vehicles=vd.vehicles)),
            OP.Routing(vd.dist, vd.demands, vd.capacity, vd.vehicles), False)


@pytest.mark.parametrize("kind", ["tsp", "knap", "cvrp"])
@pytest.mark.parametrize("T,P", SHAPES)
def test_launch_shapes_bit_identical(kind, T, P):
    prob, ref, custom = _pair(kind)
    ops = G.tsp_delta_operators() if custom else ()
    res = G.run(prob, G.EngineConfig(population=P, team_size=T, max_generations=4, seed=T + P,
                                     record_history=True, custom_operators=ops))
    out = OE.run(ref, OE.RunCfg(population=P, team_size=T, max_generations=4, seed=T + P,
                                record_history=True, allowed_ops=prob.device_sequences(),
                                custom_ops=tuple((i, nm, f, 1.0) for i, nm, f in OM.TSP_DELTA)
                                if custom else ()),
                 device_stream="philox")
    assert res.device["error_flags"] == 0
    assert res.history["best_phi"] == out.history["best_phi"]
    d1 = ref.spec.d1
    assert [[s.row(r).tolist() for r in range(d1)] for s in res.population] == \
        [[s.row(r).tolist() for r in range(d1)] for s in out.population]


@pytest.mark.parametrize("kind", ["tsp", "knap", "cvrp"])
@pytest.mark.parametrize("islands,migration,top_n", [(2, "ring", 1), (5, "ring", 1),
                                                     (3, "global_top_n", 2),
                                                     (5, "global_top_n", 3), (4, "hybrid", 2)])
def test_island_migration_sweep(kind, islands, migration, top_n):
    """engine.py:483-532: ring / global_top_n / hybrid migration every 2
    generations and elite injection every 3, uneven island sizes (P = 7)."""
    prob, ref, _ = _pair(kind)
    kw = dict(population=7, team_size=16, max_generations=9, seed=islands * 10 + top_n,
              record_history=True)
    res = G.run(prob, G.EngineConfig(islands=G.IslandsConfig(count=islands, migration=migration,
                                                             interval=2, top_n=top_n),
                                     elite_injection_interval=3, **kw))
    out = OE.run(ref, OE.RunCfg(islands=islands, migration=migration, migration_interval=2,
                                top_n=top_n, elite_interval=3,
                                allowed_ops=prob.device_sequences(), **kw),
                 device_stream="philox")
    assert res.history["best_phi"] == out.history["best_phi"]
    d1 = ref.spec.d1
    assert [[s.row(r).tolist() for r in range(d1)] for s in res.population] == \
        [[s.row(r).tolist() for r in range(d1)] for s in out.population]
