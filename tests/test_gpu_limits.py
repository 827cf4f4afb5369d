"""Sizes beyond the shared-memory fast paths (edge cases of SURVEY §8c): long
rows whose lane rows no longer fit the 227 KB opt-in shared memory run with
the lane rows in global memory (row layouts 12 / 13), and large TSP instances
read a global distance matrix — still bit-identical to the oracle."""

import numpy as np
import pytest

import paper_2603_19163_b200 as G
from oracle import engine as OE
from oracle import problems as OP
from paper_2603_19163_b200 import instances as I

pytestmark = pytest.mark.gpu


def _same(prob, ref, P, T, Gn, seed, layouts):
    res = G.run(prob, G.EngineConfig(population=P, team_size=T, max_generations=Gn, seed=seed,
                                     record_history=True))
    assert res.device["layout"] in layouts, res.device["layout"]
    out = OE.run(ref, OE.RunCfg(population=P, team_size=T, max_generations=Gn, seed=seed,
                                record_history=True, allowed_ops=prob.device_sequences()),
                 device_stream="philox")
    assert res.device["error_flags"] == 0
    assert res.history["best_phi"] == out.history["best_phi"]
    assert [s.row(0).tolist() for s in res.population] == [s.row(0).tolist() for s in out.population]


def test_knapsack_long_rows_in_global_memory():
    w, v, cap = I.knapsack_random(6000, 77)
    prob = G.builtin_problem("knapsack", G.InstanceData(weights=w, values=v, capacity=cap))
    _same(prob, OP.Knapsack(w, v, cap), 3, 64, 6, 3, (12, 13))


def test_qap_large_instance_global():
    f, d = I.qap_random(300, 5)
    prob = G.builtin_problem("qap", G.InstanceData(flow_matrix=f, distance_matrix=d))
    _same(prob, OP.Qap(f, d), 2, 32, 3, 4, (11, 12, 13))


def test_user_permutation_long_rows():
    n = 2500
    d = I.tsp_random(n, 12, True)
    tour = """
      double s = 0.0;
      for (int i = 0; i < sol.n; ++i) s += data.dist[sol[i] * sol.n + sol[i + 1 == sol.n ? 0 : i + 1]];
      return s;
    """

    def tour_py(t):
        s = 0.0
        for i in range(n):
            s += d[t[i], t[(i + 1) % n]]
        return s
    prob = G.CudaProblem("permutation", n, tour, data={"dist": d})
    ref = OP.Custom(OP.PERM, n, tour_py)
    _same(prob, ref, 2, 128, 2, 6, (12, 13))


def test_single_team_ctas_and_reused_problem():
    """A 32-lane team alone in its CTA (long rows): the lane-sort tables are
    initialised by the CTA's last thread, and a problem handle serves several
    engines in a row."""
    n = 2500
    d = I.tsp_random(n, 12, True)
    tour = "double s = 0.0; for (int i = 0; i < sol.n; ++i) " \
           "s += data.dist[sol[i] * sol.n + sol[i + 1 == sol.n ? 0 : i + 1]]; return s;"
    prob = G.CudaProblem("permutation", n, tour, data={"dist": d})
    for ops in [(0,), (1,), (2, 3)]:
        prob.device_sequences = (lambda o: lambda: o)(ops)
        r = G.run(prob, G.EngineConfig(population=2, team_size=32, max_generations=3, seed=6))
        assert r.device["error_flags"] == 0 and sorted(r.best.row(0).tolist()) == list(range(n))


def test_tsp_global_distance_matrix():
    d = I.tsp_random(1800, 21, True)
    prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=d))
    res = G.run(prob, G.EngineConfig(population=4, team_size=32, max_generations=8, seed=8,
                                     record_history=True, custom_operators=G.tsp_delta_operators()))
    assert res.device["layout"] >= 6  # the distance matrix stays in global memory (L2)
    from oracle import moves as OM
    out = OE.run(OP.Tsp(d), OE.RunCfg(population=4, team_size=32, max_generations=8, seed=8,
                                      record_history=True, allowed_ops=prob.device_sequences(),
                                      custom_ops=tuple((i, nm, f, 1.0) for i, nm, f in OM.TSP_DELTA)),
                 device_stream="philox")
    assert res.history["best_phi"] == out.history["best_phi"]
    assert res.best.row(0).tolist() == out.best.row(0).tolist()


@pytest.mark.parametrize("kind", ["qap", "knap"])
def test_float_row_instances_within_tolerance(kind):
    """Float-valued QAP / knapsack (the incremental device deltas are not the
    reference's summation order): every reported objective and penalty equals
    the oracle's evaluation of the returned solution within 1e-9 relative (the
    north star allows 1e-6)."""
    rng = np.random.default_rng(31)
    if kind == "qap":
        f, d = rng.uniform(0, 10, (40, 40)), rng.uniform(0, 10, (40, 40))
        prob = G.builtin_problem("qap", G.InstanceData(flow_matrix=f, distance_matrix=d))
        ref = OP.Qap(f, d)
    else:
        w, v = rng.uniform(1, 50, 300), rng.uniform(1, 50, 300)
        cap = float(w.sum() / 3)
        prob = G.builtin_problem("knapsack", G.InstanceData(weights=w, values=v, capacity=cap))
        ref = OP.Knapsack(w, v, cap)
    res = G.run(prob, G.EngineConfig(population=8, team_size=64, max_generations=40, seed=2))
    assert res.device["error_flags"] == 0
    for s in [res.best] + res.population:
        o = OP.Sol(s.data.copy(), s.dim2_sizes.copy(), 1)
        OP.evaluate(ref, o)
        assert s.objectives[0] == pytest.approx(o.obj[0], rel=1e-9)
        assert s.penalty == pytest.approx(o.pen, rel=1e-9, abs=1e-9)
