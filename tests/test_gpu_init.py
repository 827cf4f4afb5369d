"""Device-side population initialisation (csrc/kernels/go_init.cuh,
`EngineConfig(device_init=True)`): the random pool drawn on the device, its
evaluation and the selection equal the oracle's restatement
(`oracle.engine.init_population_philox`, engine.py:252-360 with per-solution
Philox streams) solution for solution; whole runs started from it equal the
oracle engine in Philox mode."""

import numpy as np
import pytest

import paper_2603_19163_b200 as G
from oracle import engine as OE
from oracle import problems as OP
from paper_2603_19163_b200 import engine as GE
from paper_2603_19163_b200 import instances as I

pytestmark = pytest.mark.gpu


def _pair(name):
    if name == "tsp":
        d = I.tsp_random(51, 51)
        return G.builtin_problem("tsp", G.InstanceData(distance_matrix=d)), OP.Tsp(d)
    if name == "tsp_float":
        d = I.tsp_random(40, 9, rounded=False)
        return G.builtin_problem("tsp", G.InstanceData(distance_matrix=d)), OP.Tsp(d)
    if name == "qap":
        f, d = I.qap_random(30, 100)
        return (G.builtin_problem("qap", G.InstanceData(flow_matrix=f, distance_matrix=d)),
                OP.Qap(f, d))
    if name == "knap":
        w, v, cap = I.knapsack_random(200, 1000)
        return (G.builtin_problem("knapsack", G.InstanceData(weights=w, values=v, capacity=cap)),
                OP.Knapsack(w, v, cap))
    if name == "jsp":
        jobs = I.jsp_random(6, 5, 7)
        return G.builtin_problem("jsp_int", G.InstanceData(jobs=jobs)), OP.JspInt(jobs)
    if name in ("vrptw", "cvrp"):
        vd = I.vrptw_solomon_like(n=30, vehicles=6, seed=7)
        if name == "cvrp":
            return (G.builtin_problem("cvrp", G.InstanceData(
                distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity,
                vehicles=vd.vehicles)), OP.Routing(vd.dist, vd.demands, vd.capacity, vd.vehicles))
        return (G.builtin_problem("vrptw", G.InstanceData(
            distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity,
            vehicles=vd.vehicles, ready_times=vd.ready, due_times=vd.due,
            service_times=vd.service)),
            OP.Vrptw(vd.dist, vd.demands, vd.capacity, vd.vehicles, vd.ready, vd.due,
                     vd.service))
    from tests.extra_problems import oracle_problem, product_problem
    return product_problem(name), oracle_problem(name)


def _rows(s, d1):
    return [s.row(r).tolist() for r in range(d1)]


@pytest.mark.parametrize("name", ["tsp", "tsp_float", "qap", "knap", "jsp", "vrptw", "cvrp",
                                  "assign40", "binpack30", "loadbal40", "vrpprio20",
                                  "jspperm6x4", "sched8x6"])
@pytest.mark.parametrize("pop,over,seed", [(16, 4, 42), (5, 3, 2024)])
def test_device_init_equals_oracle(name, pop, over, seed):
    prob, ref = _pair(name)
    d1 = ref.spec.d1
    got = GE.initialize_population_device(prob, pop, over, seed, 0,
                                          __import__("random").Random(0))
    want = OE.init_population_philox(ref, pop, over, seed)
    assert len(got) == len(want) == pop
    for g, w in zip(got, want):
        assert _rows(g, d1) == _rows(w, d1)
        if name == "tsp_float":  # float tours: device sum within 1e-12 relative
            assert g.objectives[0] == pytest.approx(w.obj[0], rel=1e-12)
        else:
            assert list(g.objectives) == list(w.obj) and g.penalty == w.pen


def test_device_init_multiobjective_pool_fronts():
    """Two objectives: the device draws and evaluates, the host keeps the
    non-dominated fronts (engine.py:352-360) — equal to the oracle."""
    vd = I.vrptw_solomon_like(n=20, vehicles=5, seed=3)
    names = ("distance", "vehicles")
    prob = G.builtin_problem("cvrp", G.InstanceData(
        distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity,
        vehicles=vd.vehicles, meta={"objectives": names}))
    ref = OP.Routing(vd.dist, vd.demands, vd.capacity, vd.vehicles,
                     objectives=names)
    got = GE.initialize_population_device(prob, 12, 4, 7, 0, __import__("random").Random(0))
    want = OE.init_population_philox(ref, 12, 4, 7)
    assert [_rows(g, 5) for g in got] == [_rows(w, 5) for w in want]
    assert [list(g.objectives) for g in got] == [list(w.obj) for w in want]


def test_device_init_full_size_properties():
    """C2 shape (n = 442, P = 592, 2,368 draws): every kept row is a
    permutation, the kept objectives equal a fresh device evaluation, and they
    are the pool's best in compare order (sorted, none of the dropped better)."""
    d, _ = I.tsp_lattice()
    prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=d))
    pop = GE.initialize_population_device(prob, 592, 4, 42, 0, __import__("random").Random(0))
    assert len(pop) == 592
    ident = list(range(442))
    for s in pop:
        assert sorted(s.row(0).tolist()) == ident
    objs = [s.objectives[0] for s in pop]
    assert objs == sorted(objs)
    obj, _ = G.problems.device_evaluate(prob, pop)
    assert obj[:, 0].tolist() == objs
    whole = GE.initialize_population_device(prob, 2368 + 4, 1, 42, 0,
                                            __import__("random").Random(0))
    assert len(whole) == 2372


@pytest.mark.parametrize("name,P,T,Gn,seed", [("tsp", 6, 32, 20, 5), ("knap", 4, 32, 15, 8),
                                              ("vrptw", 4, 16, 5, 9)])
def test_run_with_device_init_bit_identical_to_oracle(name, P, T, Gn, seed):
    prob, ref = _pair(name)
    res = G.run(prob, G.EngineConfig(population=P, team_size=T, max_generations=Gn, seed=seed,
                                     record_history=True, device_init=True))
    out = OE.run(ref, OE.RunCfg(population=P, team_size=T, max_generations=Gn, seed=seed,
                                record_history=True, allowed_ops=prob.device_sequences(),
                                device_init=True), device_stream="philox")
    assert res.history["best_phi"] == out.history["best_phi"]
    assert res.objectives == out.objectives and res.penalty == out.penalty
    d1 = ref.spec.d1
    assert [_rows(s, d1) for s in res.population] == [_rows(s, d1) for s in out.population]
