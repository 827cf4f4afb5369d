"""Shared builders for the further single-row built-ins (golden_extra.json)."""

import json
from pathlib import Path

import numpy as np

from oracle import problems as OP

GOLD = json.loads((Path(__file__).with_name("golden") / "golden_extra.json").read_text())


def oracle_problem(key):
    g = GOLD["instances"][key]
    name, p = g["problem"], g["payload"]
    if name == "assignment":
        return OP.Assignment(np.array(p["cost_matrix"], dtype=np.float64))
    if name == "graph_coloring":
        return OP.GraphColoring(p["meta"]["num_vertices"], p["edges"], p["num_colors"])
    if name == "bin_packing":
        return OP.BinPacking(p["item_sizes"], p["bin_capacity"])
    return OP.LoadBalancing(p["durations"], p["num_machines"])


def product_problem(key):
    import paper_2603_19163_b200 as G
    g = GOLD["instances"][key]
    kw = dict(g["payload"])
    meta = kw.pop("meta", {})
    for k in ("cost_matrix", "item_sizes", "durations"):
        if k in kw:
            kw[k] = np.asarray(kw[k], dtype=np.float64)
    return G.builtin_problem(g["problem"], G.InstanceData(meta=meta, **kw))
