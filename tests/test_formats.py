"""Instance formats, demo instances and the CLI harness on CPU.

Parsed arrays and error messages equal the reference's own parsers on the same
files (goldens from tests/golden/make_golden_formats.py); the CLI keeps the
reference's commands and exit codes (cli.py:228-249; tests/test_results_cli.py
of the reference).  Solving needs the GPU: see tests/test_gpu_cli.py."""

import json
from pathlib import Path

import numpy as np
import pytest

from paper_2603_19163_b200 import cli
from paper_2603_19163_b200 import instances as I
from paper_2603_19163_b200 import parsers as PZ
from paper_2603_19163_b200.core import Lexicographic

ROOT = Path(__file__).resolve().parents[1]
GOLD = json.loads((ROOT / "tests" / "golden" / "golden_formats.json").read_text())
PARSE = {".tsp": PZ.parse_tsplib, ".dat": PZ.parse_qaplib, ".txt": PZ.parse_solomon,
         ".jsp": PZ.parse_orlib_jsp, ".json": lambda p: PZ.parse_json_instance(p)[1]}


def _plain(v):
    if isinstance(v, np.ndarray):
        return v.tolist()
    if isinstance(v, (list, tuple)):
        return [_plain(x) for x in v]
    if isinstance(v, dict):
        return {k: _plain(x) for k, x in v.items()}
    if isinstance(v, Lexicographic):
        return {"mode": "lexicographic", "priority": list(v.priority_order),
                "tolerances": list(v.tolerances)}
    return v


@pytest.fixture(autouse=True)
def _in_repo(monkeypatch):
    monkeypatch.chdir(ROOT)  # golden paths are repo-relative, as the messages are


@pytest.mark.parametrize("name", sorted(GOLD["files"]))
def test_parsers_match_reference(name):
    g = GOLD["files"][name]
    rel = f"tests/fixtures/{name}"
    parse = PARSE[Path(name).suffix]
    if not g["ok"]:
        with pytest.raises(PZ.ParseError) as exc:
            parse(rel)
        assert str(exc.value) == g["error"] and exc.value.line == g["line"]
        return
    inst = parse(rel)
    for key, want in g["instance"].items():
        got = inst.meta if key == "meta" else getattr(inst, key)
        assert _plain(got) == want, key


def test_euclidean_distance_matrix_matches_reference():
    e = GOLD["euclid"]
    c = np.array(e["coords"])
    assert PZ.euclidean_distance_matrix(c, True).tolist() == e["rounded"]
    assert PZ.euclidean_distance_matrix(c, False).tolist() == e["exact"]


def test_demo_instances_and_generality_suite():
    demos = I.demo_instances()
    assert len(demos) == 13 and set(I.GENERALITY_SUITE) <= set(demos)
    assert demos["tsp4"].best_known == 14.0 and demos["vrptw8"].best_known is None
    assert I.demo_instance("qap5").problem_name == "qap"
    with pytest.raises(ValueError):
        I.demo_instance("nope")
    d = I.cvrp8_instance().distance_matrix  # chain clusters (instances.py:32-47, :170-184)
    assert d[0, 1] == 20.0 and d[0, 2] == 45.0 and d[1, 4] == 45.0 and d[1, 5] == 60.0


def _cli(capsys, *argv):
    rc = cli.main(list(argv))
    out = capsys.readouterr()
    return rc, out.out, out.err


def test_cli_commands_and_exit_codes(capsys):
    rc, out, _ = _cli(capsys, "list-problems")
    assert rc == 0 and "demo:tsp5" in out and "schedule_binary" in out and "tsp-delta" in out
    rc, out, _ = _cli(capsys, "validate", "--instance", "demo:cvrp10")
    assert rc == 0 and out.strip() == "cvrp10: problem=cvrp encoding=permutation d1=4 d2=10 n=10"
    rc, out, _ = _cli(capsys, "validate", "--problem", "tsp", "--instance",
                      "tests/fixtures/euc17.tsp")
    assert rc == 0 and "d2=17" in out
    rc, out, _ = _cli(capsys, "validate", "--instance", "tests/fixtures/knap.json")
    assert rc == 0 and "problem=knapsack encoding=binary" in out
    # usage errors: 1
    for argv in (["solve"], ["bogus"], ["validate", "--instance", "x.tsp"],
                 ["validate", "--problem", "knapsack", "--instance", "x.txt"],
                 ["validate", "--problem", "qap", "--instance", "demo:tsp4"],
                 ["bench", "--instance", "demo:tsp4", "--seeds", ","]):
        rc, _, err = _cli(capsys, *argv)
        assert rc == 1 and err.startswith("usage error:"), argv
    # parse errors: 2
    rc, _, err = _cli(capsys, "validate", "--problem", "tsp", "--instance",
                      "tests/fixtures/short.tsp")
    assert rc == 2 and err.strip() == "parse error: " + GOLD["files"]["short.tsp"]["error"]
    rc, _, _ = _cli(capsys, "validate", "--problem", "tsp", "--instance", "tests/fixtures/nah.tsp")
    assert rc == 2
    # other errors: 3 (unknown demo)
    rc, _, err = _cli(capsys, "validate", "--instance", "demo:nope")
    assert rc == 3 and err.startswith("error:")


def test_cli_engine_config_mapping():
    args = cli.build_parser().parse_args(
        ["solve", "--instance", "demo:tsp5", "--pop", "8", "--team-size", "16", "--islands", "2",
         "--migration", "hybrid", "--aos-interval", "5", "--custom-ops", "tsp-delta",
         "--fast-budget", "4096", "--device-init", "--target", "18"])
    cfg = cli.engine_config_from_args(args, 7)
    assert (cfg.population, cfg.team_size, cfg.seed, cfg.islands.count) == (8, 16, 7, 2)
    assert cfg.islands.migration == "hybrid" and cfg.aos.update_interval == 5
    assert [op.name for op in cfg.custom_operators] == \
        ["delta_two_opt", "delta_or_opt", "delta_node_insert"]
    assert cfg.fast_budget_bytes == 4096 and cfg.device_init and cfg.target_objective == 18


@pytest.mark.parametrize("name", ["euc17.tsp", "upper9.tsp", "full9.tsp", "qap7.dat", "sol12.txt",
                                  "js5x4.jsp"])
def test_truncation_fuzz_raises_positioned_errors(name, tmp_path):
    """Reference acceptance criterion 10 (test_acceptance.py:313-343): every
    prefix of a valid file either parses or raises ParseError — never another
    exception."""
    raw = (ROOT / "tests" / "fixtures" / name).read_bytes()
    parse = PARSE[Path(name).suffix]
    step = max(1, len(raw) // 40)
    for cut in range(0, len(raw), step):
        stub = tmp_path / name
        stub.write_bytes(raw[:cut])
        try:
            parse(str(stub))
        except PZ.ParseError as exc:
            assert str(stub) in str(exc)


def test_parsed_matrices_are_symmetric_nonnegative():
    for name, parse in (("euc17.tsp", PZ.parse_tsplib), ("upper9.tsp", PZ.parse_tsplib),
                        ("sol12.txt", PZ.parse_solomon)):
        d = parse(str(ROOT / "tests" / "fixtures" / name)).distance_matrix
        assert np.array_equal(d, d.T) and not np.any(np.diag(d)) and np.all(d >= 0)
