"""The gap references of bench.py (tools/bounds.py, profiles/best_known.json):
exact knapsack optimum against brute force, the 1-tree bound below known
tours, the JSP bound below schedules, and the stored table consistent with
them."""
import importlib.util
import itertools
import json
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
spec = importlib.util.spec_from_file_location("bounds", ROOT / "tools" / "bounds.py")
B = importlib.util.module_from_spec(spec)
spec.loader.exec_module(B)


def test_knapsack_dp_matches_brute_force():
    rng = np.random.default_rng(5)
    for _ in range(5):
        w = rng.integers(1, 30, 12)
        v = rng.integers(1, 50, 12)
        cap = int(w.sum() // 2)
        best = max(sum(v[list(s)]) for k in range(13) for s in itertools.combinations(range(12), k)
                   if sum(w[list(s)]) <= cap)
        assert B.knapsack_optimum(w, v, cap) == best


def test_one_tree_bound_below_the_lattice_optimum():
    from paper_2603_19163_b200 import instances as I
    d, opt = I.tsp_lattice(cols=6, rows=4)
    lb = B.one_tree_bound(d, upper=opt * 1.05, iters=400)
    assert lb <= opt + 1e-6 and lb >= 0.9 * opt


def test_best_known_table_is_consistent():
    bk = json.loads((ROOT / "profiles" / "best_known.json").read_text())
    assert bk["C5b"]["best_known"] <= bk["C5b"]["optimum"] and bk["C5b"]["sense"] == "max"
    assert bk["C2j"]["lower_bound"] <= bk["C2j"]["best_known"]
    assert bk["C5a"]["lower_bound"] <= bk["C5a"]["best_known"]
    assert bk["C2"]["optimum"] == 44200.0
    assert bk["C3"]["penalty_lower_bound"] > 8.0  # R101: lateness no route avoids
