"""CLI harness and the reference's generality criterion on the B200 engine
(reference tests/test_results_cli.py and
tests/test_acceptance.py:88-115): `solve` / `bench` documents through
`ResultRecord`, and every demo instance of GENERALITY_SUITE that has a device
path reaches its oracle-verified optimum on 5/5 seeds with the reference's
settings (population 8, team 8, <= 2000 generations, target = optimum)."""

import json
from pathlib import Path

import pytest

import paper_2603_19163_b200 as G
from paper_2603_19163_b200 import cli
from paper_2603_19163_b200 import instances as I
from paper_2603_19163_b200.problems import DEVICE_PROBLEMS
from paper_2603_19163_b200.results import RESULT_SCHEMA_FIELDS, parse_results

pytestmark = pytest.mark.gpu
SEEDS = (42, 123, 456, 789, 2024)  # reference tests/test_acceptance.py:41


def test_cli_solve_and_bench_documents(tmp_path, capsys):
    root = Path(__file__).resolve().parents[1]
    out = tmp_path / "r.json"
    assert cli.main(["solve", "--instance", "demo:tsp5", "--pop", "8", "--team-size", "8",
                     "--generations", "300", "--seed", "7", "--json", str(out)]) == 0
    doc = json.loads(out.read_text())
    assert list(doc) == list(RESULT_SCHEMA_FIELDS)
    assert doc["problem"] == "tsp" and doc["instance"] == "tsp5" and doc["seed"] == 7
    assert doc["objectives"] == [18.0] and doc["gap_pct"] == 0.0 and doc["feasible"]
    rc = cli.main(["bench", "--instance", "demo:tsp4", "--instance",
                   str(root / "tests/fixtures/knap.json"), "--seeds", "1,2", "--pop", "4",
                   "--team-size", "8", "--generations", "50", "--device-init"])
    cap = capsys.readouterr()
    assert rc == 0
    recs = parse_results(cap.out)
    assert [(r.instance, r.seed) for r in recs] == [("tsp4", 1), ("tsp4", 2), ("knap.json", 1),
                                                    ("knap.json", 2)]
    assert recs[0].objectives == [14.0] and recs[2].objectives == [9.0]
    assert "tsp4" in cap.err  # gap table on stderr when stdout carries the documents
    rc = cli.main(["solve", "--problem", "tsp", "--instance", str(root / "tests/fixtures/euc17.tsp"),
                   "--generations", "100", "--pop", "8", "--team-size", "32"])
    cap = capsys.readouterr()
    assert rc == 0 and json.loads(cap.out)["instance"] == "euc17.tsp"
    # MULTI_FIXED rows (binary worker x shift schedule) through the same CLI
    rc = cli.main(["solve", "--instance", "demo:schedule3x4", "--pop", "8", "--team-size", "8",
                   "--generations", "500", "--target", "21"])
    cap = capsys.readouterr()
    assert rc == 0 and json.loads(cap.out)["objectives"] == [21.0]
    rc = cli.main(["solve", "--instance", "demo:nope"])
    assert rc == 3 and "unknown demo instance" in capsys.readouterr().err


@pytest.mark.parametrize("name", [n for n in I.GENERALITY_SUITE])
def test_generality_suite_reaches_optima(name):
    demo = I.demo_instance(name)
    if demo.problem_name not in DEVICE_PROBLEMS:
        pytest.skip(f"{demo.problem_name} has no device path in this build")
    prob = demo.problem()
    if demo.best_known is None:  # vrptw8: feasibility + the same value on every seed
        vals = []
        for seed in SEEDS:
            r = G.run(prob, G.EngineConfig(population=8, team_size=8, max_generations=300,
                                           seed=seed))
            assert r.feasible, seed
            vals.append(r.objectives[0])
        assert len(set(vals)) == 1, vals
        return
    for seed in SEEDS:
        r = G.run(prob, G.EngineConfig(population=8, team_size=8, max_generations=2000,
                                       seed=seed, target_objective=demo.best_known),
                  best_known=demo.best_known)
        assert r.feasible and r.generations_completed <= 2000, seed
        assert r.objectives[0] == pytest.approx(demo.best_known, abs=1e-9), (seed, r.objectives)
