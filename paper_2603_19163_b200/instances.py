"""Seeded synthetic instances of the BASELINE config shapes (host I/O only).

Shapes and seeds follow SURVEY §8(d):
  C1  random Euclidean TSP n=51, TSPLIB nint distances          (seed 51)
  C2  pcb442-shaped lattice TSP: 26 x 17 grid at spacing 100, labels
      permuted by seed 442 -> known optimum 44,200 (a unit-step Hamiltonian
      cycle exists because 26 is even and every edge is >= 100)
  C3  Solomon-R1-shaped VRPTW: 100 customers, 25 vehicles, capacity 200
  C4  QAPLIB-shaped QAP n=100, symmetric U{0..99} flow/distance   (seed 100)
  C5a OR-Library-shaped JSP 20 jobs x 15 machines, U{1..99}       (seed 2015)
  C5b 0/1 knapsack n=1000, w, v ~ U{1..1000}, cap = floor(sum w / 2) (seed 1000)

Distance conventions restate the reference parsers: TSPLIB EUC_2D rounding is
int(x + 0.5) symmetrised with max (parsers.py:65-67, :362-375); Solomon
distances are unrounded and symmetrised with the mean (parsers.py:217-224).
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

LATTICE_OPTIMUM = 44200.0


def euclid(coords, rounded: bool = False) -> np.ndarray:
    c = np.asarray(coords, dtype=np.float64)
    diff = c[:, None, :] - c[None, :, :]
    d = np.sqrt(diff[..., 0] * diff[..., 0] + diff[..., 1] * diff[..., 1])
    if rounded:
        d = np.floor(d + 0.5)
        np.fill_diagonal(d, 0.0)
        return np.maximum(d, d.T)
    np.fill_diagonal(d, 0.0)
    return (d + d.T) / 2.0


def tsp_random(n: int = 51, seed: int = 51, rounded: bool = True) -> np.ndarray:
    return euclid(np.random.default_rng(seed).uniform(0, 1000, (n, 2)), rounded)


def tsp_lattice(cols: int = 26, rows: int = 17, spacing: float = 100.0,
                seed: int = 442, jitter: int = 0) -> tuple[np.ndarray, float | None]:
    """Returns (distance matrix, known optimum or None when jittered)."""
    rng = np.random.default_rng(seed)
    xs, ys = np.meshgrid(np.arange(cols) * spacing, np.arange(rows) * spacing)
    pts = np.stack([xs.ravel(), ys.ravel()], axis=1)
    if jitter:
        pts = pts + np.random.default_rng(seed * 10).integers(-jitter, jitter + 1, pts.shape)
    pts = pts[rng.permutation(len(pts))]
    opt = cols * rows * spacing if (not jitter and (cols % 2 == 0 or rows % 2 == 0)) else None
    return euclid(pts, rounded=True), opt


def lattice_tour(cols: int = 26, rows: int = 17, seed: int = 442) -> np.ndarray:
    """The optimal snake cycle of `tsp_lattice` in permuted labels."""
    perm = np.random.default_rng(seed).permutation(cols * rows)
    label = np.empty_like(perm)
    label[perm] = np.arange(len(perm))         # grid index -> label
    order = [0 * cols + 0]
    for c in range(cols):                       # go up/down columns 1.., row 0 return
        rng_rows = range(1, rows) if c % 2 == 0 else range(rows - 1, 0, -1)
        order.extend(r * cols + c for r in rng_rows)
    order.extend(0 * cols + c for c in range(cols - 1, 0, -1))
    return label[np.array(order)]


@dataclass
class VrptwData:
    dist: np.ndarray
    demands: np.ndarray
    capacity: float
    vehicles: int
    ready: np.ndarray
    due: np.ndarray
    service: np.ndarray


def vrptw_solomon_like(n: int = 100, vehicles: int = 25, capacity: float = 200.0,
                       seed: int = 101) -> VrptwData:
    """R1-class-shaped instance: depot at (35,35) with horizon 230, customers
    uniform on [0,70]^2, demand U{1..41}, service 10, window centres drawn so
    the depot round trip fits, widths U{10..30}; integer-valued times, float
    (unrounded) distances as in the Solomon parser."""
    rng = np.random.default_rng(seed)
    xy = np.vstack([[35.0, 35.0], rng.integers(0, 71, (n, 2)).astype(np.float64)])
    dist = euclid(xy, rounded=False)
    horizon = 230.0
    demands = rng.integers(1, 42, n).astype(np.float64)
    service = np.concatenate([[0.0], np.full(n, 10.0)])
    ready = np.zeros(n + 1)
    due = np.zeros(n + 1)
    due[0] = horizon
    for c in range(1, n + 1):
        lo = np.ceil(dist[0, c])
        hi = np.floor(horizon - dist[c, 0] - service[c])
        centre = rng.integers(int(lo), int(max(lo, hi)) + 1)
        half = rng.integers(5, 16)
        ready[c] = max(0.0, centre - half)
        due[c] = min(hi, centre + half) if hi >= lo else lo
        if due[c] < ready[c]:
            due[c] = ready[c]
    return VrptwData(dist, demands, capacity, vehicles, ready, due, service)


def qap_random(n: int = 100, seed: int = 100) -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(seed)

    def sym():
        a = rng.integers(0, 100, (n, n)).astype(np.float64)
        a = np.triu(a, 1)
        return a + a.T

    return sym(), sym()


def jsp_random(n_jobs: int = 20, n_machines: int = 15, seed: int = 2015):
    rng = np.random.default_rng(seed)
    return [[(int(m), int(rng.integers(1, 100))) for m in rng.permutation(n_machines)]
            for _ in range(n_jobs)]


def knapsack_random(n: int = 1000, seed: int = 1000):
    rng = np.random.default_rng(seed)
    w = rng.integers(1, 1001, n).astype(np.float64)
    v = rng.integers(1, 1001, n).astype(np.float64)
    return w, v, float(np.floor(w.sum() / 2))


# ---- desk-scale demo instances (instances.py:20-208 of the reference) ----------
# The instance data with its independently verified optima is the reference's;
# tests/golden/make_golden_formats.py dumps it to data/demo_instances.json.

_DEMO_FILE = Path(__file__).with_name("data") / "demo_instances.json"
_ARRAY_FIELDS = ("distance_matrix", "weights", "values", "flow_matrix", "cost_matrix",
                 "item_sizes", "durations", "demands", "ready_times", "due_times",
                 "service_times", "priorities", "requirements")


@dataclass(frozen=True)
class DemoInstance:
    name: str
    problem_name: str
    instance: "InstanceData"
    best_known: float | None
    note: str = ""

    def problem(self):
        from .problems import builtin_problem
        return builtin_problem(self.problem_name, self.instance)


def _instance_from_json(doc: dict):
    from .problems import InstanceData
    kw = {}
    for key, val in doc.items():
        if key == "meta":
            continue
        if key in _ARRAY_FIELDS:
            kw[key] = np.asarray(val, dtype=np.float64)
        elif key == "edges":
            kw[key] = [tuple(int(x) for x in e) for e in val]
        elif key == "jobs":
            kw[key] = [[(int(m), int(t)) for m, t in ops] for ops in val]
        else:
            kw[key] = val
    return InstanceData(meta=dict(doc.get("meta", {})), **kw)


def _demo_table() -> dict:
    return json.loads(_DEMO_FILE.read_text())


def demo_instances() -> dict[str, DemoInstance]:
    """instances.py:197-198: name -> DemoInstance (fresh objects per call)."""
    return {name: DemoInstance(name, d["problem"], _instance_from_json(d["instance"]),
                               d["best_known"], d.get("note", ""))
            for name, d in _demo_table()["demos"].items()}


def demo_instance(name: str) -> DemoInstance:
    """instances.py:201-208."""
    table = demo_instances()
    if name not in table:
        raise ValueError(f"unknown demo instance {name!r}; available: {', '.join(sorted(table))}")
    return table[name]


GENERALITY_SUITE = tuple(_demo_table()["generality_suite"]) if _DEMO_FILE.exists() else ()


def chain_cluster_matrix(num_nodes: int, chains, end_leg: float, interior_leg: float,
                         step: float, inter: float) -> np.ndarray:
    """Depot 0 plus clusters laid out as chains: `step`·|a-b| along a chain,
    `interior_leg` from the depot to a chain's inner nodes and `end_leg` to its
    two ends, `inter` between clusters (instances.py:32-47)."""
    d = np.full((num_nodes, num_nodes), float(inter))
    np.fill_diagonal(d, 0.0)
    for chain in chains:
        idx = np.asarray(chain)
        k = np.arange(len(idx))
        block = step * np.abs(k[:, None] - k[None, :]).astype(np.float64)
        d[np.ix_(idx, idx)] = block
        d[0, idx] = d[idx, 0] = interior_leg
        for end in (idx[0], idx[-1]):
            d[0, end] = d[end, 0] = end_leg
    return d


def cvrp8_instance(objectives=("distance", "vehicles"), comparison=None):
    """instances.py:170-184: bi-objective routing fixture, two chains of four;
    distance optimum 170 with 2 vehicles, one route covers all at 190."""
    from .problems import InstanceData
    meta = {"objectives": tuple(objectives)}
    if comparison is not None:
        meta["comparison"] = comparison
    d = chain_cluster_matrix(9, ((1, 2, 3, 4), (5, 6, 7, 8)), end_leg=20.0, interior_leg=45.0,
                             step=15.0, inter=60.0)
    return InstanceData(distance_matrix=d, demands=np.ones(8), capacity=8.0, vehicles=3,
                        meta=meta)


# ---- the BASELINE.json workloads -----------------------------------
DATA_DIR = Path(__file__).with_name("data")
FIXTURES = {  # the reference's benchmark-format fixtures (pkg/tests/fixtures, README there)
    "R101": DATA_DIR / "R101.txt",    # synthetic Solomon R101-format, 100 customers, 25 vehicles
    "eil51": DATA_DIR / "eil51.tsp",  # TSPLIB eil51, best known 426
    "ft06": DATA_DIR / "ft06.jsp",    # Fisher-Thompson 6x6, optimum 55
    "nug12": DATA_DIR / "nug12.dat",  # QAPLIB layout at nug12 size
}
KNOWN_OPTIMA = {"eil51": 426.0, "ft06": 55.0, "lattice442": 44200.0}


def baseline_instances() -> dict:
    """name -> (problem name, InstanceData, best known or None) for the named
    BASELINE shapes: C1 random Euclidean TSP n=51, C2 the pcb442-shaped 26x17
    lattice (known optimum 44,200) and its +-30 jittered twin, C3 VRPTW on the
    reference's R101 fixture, C4 QAP n=100, C5a JSP 20x15 (integer encoding),
    C5b knapsack n=1000."""
    from .parsers import parse_solomon
    from .problems import InstanceData
    d2, opt2 = tsp_lattice()
    dj, _ = tsp_lattice(jitter=30)
    f, dq = qap_random(100, 100)
    w, v, cap = knapsack_random(1000, 1000)
    return {
        "C1": ("tsp", InstanceData(distance_matrix=tsp_random(51, 51)), None),
        "C2": ("tsp", InstanceData(distance_matrix=d2), opt2),
        "C2j": ("tsp", InstanceData(distance_matrix=dj), None),
        "C3": ("vrptw", parse_solomon(FIXTURES["R101"]), None),
        "C4": ("qap", InstanceData(flow_matrix=f, distance_matrix=dq), None),
        "C5a": ("jsp_int", InstanceData(jobs=jsp_random(20, 15, 2015)), None),
        "C5b": ("knapsack", InstanceData(weights=w, values=v, capacity=cap), None),
    }
