"""Bit-exact parity at the exact launch shapes bench.py measures (VERDICT r1
"Next" #1): the B200 population rule picks P (one resident wave, e.g. C2:
148 SMs x 3 teams = 444 evolvers of 128 lanes on 148 co-resident cooperative
CTAs, crossover mates waited on across CTAs), the full reference registry
(+ tsp-delta user operators on C2), and a few generations are compared with
the Philox-mode oracle: per-generation best-Φ history, final population,
best solution, AOS weights.  The oracle evolves each generation's evolvers in
parallel host processes (oracle.engine.run(workers=...)), identical to the
serial loop."""
import os

import pytest

import paper_2603_19163_b200 as G
from oracle import engine as OE
from tests.helpers import bench_pairs

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

GENS = {"C1": 3, "C2": 3, "C3": 2, "C4": 2, "C5a": 2, "C5b": 3}


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5a", "C5b"])
def test_bench_launch_shape_bit_identical(name):
    prob, ref, ops, oops = bench_pairs((name,))[name]
    gens = GENS[name]
    res = G.run(prob, G.EngineConfig(team_size=128, seed=42, custom_operators=ops,
                                     max_generations=gens, record_history=True))
    P = res.config["population_effective"]
    dr_sm = G._native.device_info(0).sm_count
    assert P % dr_sm == 0 and P >= dr_sm  # one resident wave of whole SMs, as bench.py runs
    workers = max(1, min(32, len(os.sched_getaffinity(0))))
    out = OE.run(ref, OE.RunCfg(population=P, team_size=128, max_generations=gens, seed=42,
                                record_history=True, allowed_ops=prob.device_sequences(),
                                custom_ops=oops),
                 device_stream="philox", workers=workers)
    assert res.device["error_flags"] == 0
    assert res.generations_completed == out.generations == gens
    assert [e["id"] for e in res.final_weights["sequences"]] == out.ids
    assert res.history["best_phi"] == out.history["best_phi"]
    assert res.objectives == out.objectives and res.penalty == out.penalty
    assert _cells(res.best.data, res.best.dim2_sizes) == _cells(out.best.data, out.best.sizes)
    assert [e["weight"] for e in res.final_weights["sequences"]] == [float(w) for w in out.weights]
    # active cells row by row (cells past a row's size are not part of a solution)
    assert [_cells(s.data, s.dim2_sizes) for s in res.population] == \
        [_cells(s.data, s.sizes) for s in out.population]


def _cells(data, sizes):
    return [list(map(int, row[:int(k)])) for row, k in zip(data, sizes)]
