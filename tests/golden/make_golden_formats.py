"""Fixtures and goldens for the instance formats and the CLI,
from the UNMODIFIED reference (build container only).

    PYTHONPATH=/root/repo python tests/golden/make_golden_formats.py

1. Writes our own seeded instance files under tests/fixtures/ (TSPLIB EUC_2D and
   EXPLICIT, QAPLIB, Solomon, OR-Library JSP, JSON payloads) plus malformed
   variants, parses each with the reference's parsers (parsers.py:65-359) and
   freezes the parsed arrays or the ParseError message in golden_formats.json.
2. Dumps the reference's demo instances (instances.py:50-208) to
   paper_2603_19163_b200/data/demo_instances.json, the data file the package's
   `instances.demo_instances()` serves to the CLI.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
ROOT = Path(__file__).resolve().parents[2]

import genopt.parsers as RP  # noqa: E402
from genopt.core import Lexicographic, Weighted  # noqa: E402
from genopt.instances import GENERALITY_SUITE, demo_instances  # noqa: E402

FIX = ROOT / "tests" / "fixtures"
OUT = Path(__file__).with_name("golden_formats.json")
DEMO = ROOT / "paper_2603_19163_b200" / "data" / "demo_instances.json"

FIELDS = ("distance_matrix", "weights", "values", "capacity", "flow_matrix", "cost_matrix",
          "edges", "num_colors", "item_sizes", "bin_capacity", "durations", "num_machines",
          "jobs", "demands", "vehicles", "ready_times", "due_times", "service_times",
          "priorities", "requirements")


def plain(x):
    if isinstance(x, np.ndarray):
        return x.tolist()
    if isinstance(x, (np.floating, np.integer)):
        return x.item()
    if isinstance(x, (list, tuple)):
        return [plain(v) for v in x]
    if isinstance(x, dict):
        return {k: plain(v) for k, v in x.items()}
    if isinstance(x, Weighted):
        return {"mode": "weighted", "weights": list(x.weights)}
    if isinstance(x, Lexicographic):
        return {"mode": "lexicographic", "priority": list(x.priority_order),
                "tolerances": list(x.tolerances)}
    return x


def dump(inst):
    out = {f: plain(getattr(inst, f)) for f in FIELDS if getattr(inst, f) is not None}
    out["meta"] = plain(inst.meta or {})
    return out


def fixtures():
    rng = np.random.default_rng(2603)
    files = {}
    # TSPLIB EUC_2D (with an EOF sentinel and a comment header)
    pts = rng.uniform(0, 500, size=(17, 2)).round(2)
    body = "\n".join(f"{i + 1} {x} {y}" for i, (x, y) in enumerate(pts))
    files["euc17.tsp"] = ("tsp", "NAME : euc17\nCOMMENT : seeded fixture\nTYPE : TSP\n"
                                 f"DIMENSION : 17\nEDGE_WEIGHT_TYPE : EUC_2D\n"
                                 f"NODE_COORD_SECTION\n{body}\nEOF\n")
    m = rng.integers(1, 90, size=(9, 9))
    m = np.triu(m, 1)
    m = m + m.T
    upper = "\n".join(" ".join(str(m[i, j]) for j in range(i + 1, 9)) for i in range(8))
    files["upper9.tsp"] = ("tsp", "NAME: upper9\nTYPE: TSP\nDIMENSION: 9\n"
                                  "EDGE_WEIGHT_TYPE: EXPLICIT\nEDGE_WEIGHT_FORMAT: UPPER_ROW\n"
                                  f"EDGE_WEIGHT_SECTION\n{upper}\nEOF\n")
    full = "\n".join(" ".join(str(v) for v in row) for row in m)
    files["full9.tsp"] = ("tsp", "DIMENSION: 9\nEDGE_WEIGHT_TYPE: EXPLICIT\n"
                                 f"EDGE_WEIGHT_FORMAT: FULL_MATRIX\nEDGE_WEIGHT_SECTION\n{full}\n")
    asym = m.copy()
    asym[0, 1] += 1
    files["asym.tsp"] = ("tsp", "DIMENSION: 9\nEDGE_WEIGHT_TYPE: EXPLICIT\n"
                                "EDGE_WEIGHT_FORMAT: FULL_MATRIX\nEDGE_WEIGHT_SECTION\n" +
                         "\n".join(" ".join(str(v) for v in row) for row in asym) + "\n")
    files["nodim.tsp"] = ("tsp", "NAME: x\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n1 0 0\n")
    files["baddim.tsp"] = ("tsp", "DIMENSION: many\nEDGE_WEIGHT_TYPE: EUC_2D\n")
    files["geo.tsp"] = ("tsp", "DIMENSION: 3\nEDGE_WEIGHT_TYPE: GEO\nNODE_COORD_SECTION\n"
                               "1 0 0\n2 1 1\n3 2 2\n")
    files["short.tsp"] = ("tsp", "DIMENSION: 4\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n"
                                 "1 0 0\n2 3 4\n3 6\n")
    files["letters.tsp"] = ("tsp", "DIMENSION: 2\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n"
                                   "1 0 0\n2 x 4\n")
    # QAPLIB
    n = 7
    f = rng.integers(0, 10, size=(n, n))
    d = rng.integers(0, 10, size=(n, n))
    files["qap7.dat"] = ("qap", f"{n}\n\n" + "\n".join(" ".join(map(str, r)) for r in f) +
                         "\n\n" + "\n".join(" ".join(map(str, r)) for r in d) + "\n")
    files["qap_trunc.dat"] = ("qap", "3\n1 2 3\n4 5 6\n7 8 9\n0 1\n")
    # Solomon
    rows = []
    for cid in range(13):
        x, y = rng.integers(0, 60, size=2)
        rows.append((cid, int(x), int(y), 0 if cid == 0 else int(rng.integers(1, 20)),
                     int(rng.integers(0, 50)), int(rng.integers(100, 200)), 0 if cid == 0 else 10))
    order = [0] + list(rng.permutation(np.arange(1, 13)))  # rows out of id order
    table = "\n".join("  ".join(str(v) for v in rows[i]) for i in order)
    files["sol12.txt"] = ("vrptw", "S12\n\nVEHICLE\nNUMBER     CAPACITY\n  4         60\n\n"
                                   "CUSTOMER\nCUST NO.  XCOORD.  YCOORD.  DEMAND  READY TIME  "
                                   f"DUE DATE  SERVICE TIME\n\n{table}\n")
    files["sol_noveh.txt"] = ("vrptw", "CUSTOMER\n0 1 1 0 0 100 0\n")
    # OR-Library job shop
    jobs = [[(int(mm), int(rng.integers(1, 30))) for mm in rng.permutation(4)] for _ in range(5)]
    files["js5x4.jsp"] = ("jsp_int", "instance js5x4\n+++\nseeded fixture\n 5 4\n" +
                          "\n".join(" ".join(f"{mm} {dd}" for mm, dd in ops) for ops in jobs) + "\n")
    files["js_badm.jsp"] = ("jsp_int", "2 2\n0 3 5 4\n1 2 0 1\n")
    # JSON payloads
    files["knap.json"] = ("knapsack", json.dumps({"problem": "knapsack", "weights": [3, 4, 5],
                                                  "values": [4, 5, 6], "capacity": 7}))
    files["cvrp_mo.json"] = ("cvrp", json.dumps({
        "problem": "cvrp", "dist": (np.arange(16).reshape(4, 4) % 5).tolist(),
        "demands": [1, 2, 1], "capacity": 3, "vehicles": 2,
        "objectives": ["distance", "vehicles"],
        "comparison": {"mode": "lexicographic", "priority": [1, 0], "tolerances": [0, 0.5]}}))
    files["gc.json"] = ("graph_coloring", json.dumps({"problem": "graph_coloring",
                                                      "edges": [[0, 1], [1, 2]], "colors": 2}))
    files["nokey.json"] = ("tsp", json.dumps({"dist": [[0, 1], [1, 0]]}))
    files["badjson.json"] = ("tsp", "{not json")
    files["badmode.json"] = ("tsp", json.dumps({"problem": "tsp", "dist": [[0, 1], [1, 0]],
                                                "comparison": {"mode": "pareto"}}))
    return files


PARSERS = {".tsp": RP.parse_tsplib, ".dat": RP.parse_qaplib, ".txt": RP.parse_solomon,
           ".jsp": RP.parse_orlib_jsp, ".json": lambda p: RP.parse_json_instance(p)[1]}


def main():
    FIX.mkdir(parents=True, exist_ok=True)
    gold = {"files": {}}
    for name, (problem, text) in fixtures().items():
        path = FIX / name
        path.write_text(text)
        rel = f"tests/fixtures/{name}"
        try:
            inst = PARSERS[path.suffix](rel)
            gold["files"][name] = {"problem": problem, "ok": True, "instance": dump(inst)}
        except RP.ParseError as exc:
            gold["files"][name] = {"problem": problem, "ok": False, "error": str(exc),
                                   "line": exc.line}
    coords = np.random.default_rng(5).uniform(0, 100, size=(12, 2))
    gold["euclid"] = {"coords": coords.tolist(),
                      "rounded": RP.euclidean_distance_matrix(coords, True).tolist(),
                      "exact": RP.euclidean_distance_matrix(coords, False).tolist()}
    OUT.write_text(json.dumps(gold, indent=1))
    demos = {name: {"problem": d.problem_name, "best_known": d.best_known, "note": d.note,
                    "instance": dump(d.instance)} for name, d in demo_instances().items()}
    DEMO.parent.mkdir(parents=True, exist_ok=True)
    DEMO.write_text(json.dumps({"generality_suite": list(GENERALITY_SUITE), "demos": demos},
                               indent=1))
    print(f"{len(gold['files'])} fixture files, {len(demos)} demo instances")


if __name__ == "__main__":
    main()
