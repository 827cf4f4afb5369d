"""Shared builders for the further built-ins (golden_extra.json)."""

import json
from pathlib import Path

import numpy as np

from oracle import problems as OP

GOLD = json.loads((Path(__file__).with_name("golden") / "golden_extra.json").read_text())


def sol_rows(rows, d2):
    """(data d1 x d2 zero-padded, sizes) from a list of active rows."""
    data = np.zeros((len(rows), d2), dtype=np.int64)
    for r, row in enumerate(rows):
        data[r, :len(row)] = row
    return data, np.array([len(row) for row in rows])


def oracle_problem(key):
    g = GOLD["instances"][key]
    name, p = g["problem"], g["payload"]
    if name in ("vrp_priority", "vrp_nonlinear"):
        d = np.array(p["distance_matrix"], dtype=np.float64)
        if name == "vrp_priority":
            return OP.PriorityVrp(d, p["demands"], p["capacity"], p["vehicles"], p["priorities"])
        return OP.NonlinearVrp(d, p["demands"], p["capacity"], p["vehicles"])
    if name == "jsp_perm":
        return OP.JspPerm(p["jobs"])
    if name == "schedule_binary":
        return OP.BinarySchedule(p["cost_matrix"], p["requirements"])
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
    for k in ("cost_matrix", "item_sizes", "durations", "distance_matrix", "demands", "priorities",
              "requirements"):
        if k in kw:
            kw[k] = np.asarray(kw[k], dtype=np.float64)
    if "jobs" in kw:
        kw["jobs"] = [[tuple(op) for op in ops] for ops in kw["jobs"]]
    return G.builtin_problem(g["problem"], G.InstanceData(meta=meta, **kw))
