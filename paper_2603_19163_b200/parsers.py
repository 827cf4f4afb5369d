"""Instance file formats feeding the engine (host I/O).

API mirror of the reference's `parsers.py`: TSPLIB EUC_2D / EXPLICIT
(:65-146), QAPLIB (:149-162), Solomon VRPTW (:165-234), OR-Library job shop
(:237-274), JSON payload documents (:277-359) and `euclidean_distance_matrix`
(:362-375).  Every parser returns an `InstanceData` and raises `ParseError`
("<path>:<line>: <message>") on malformed or truncated input; the parsed
numbers equal the reference's (tests/test_formats.py against goldens made by
tests/golden/make_golden_formats.py from the reference's own parsers)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .core import Lexicographic, Weighted
from .problems import InstanceData


class ParseError(ValueError):
    """parsers.py:18-23 — carries the file and (when known) the 1-based line."""

    def __init__(self, path, message, line: int | None = None):
        self.path = str(path)
        self.line = line
        where = self.path if line is None else f"{self.path}:{line}"
        super().__init__(f"{where}: {message}")


def _lines_of(path) -> list[str]:
    try:
        return Path(path).read_text().splitlines()
    except OSError as exc:
        raise ParseError(path, f"cannot read file ({exc})") from exc


class _Scanner:
    """Numbers from whitespace-separated tokens starting at a line; a bare
    `EOF` token ends the stream (TSPLIB).  Positions are kept for errors."""

    def __init__(self, path, lines, first: int = 0):
        self.path = path
        self.toks: list[tuple[str, int]] = []
        self.pos = 0
        for idx in range(first, len(lines)):
            words = lines[idx].split()
            if "EOF" in words:
                self.toks += [(w, idx + 1) for w in words[:words.index("EOF")]]
                return
            self.toks += [(w, idx + 1) for w in words]

    def remaining(self) -> int:
        return len(self.toks) - self.pos

    def number(self, what: str) -> float:
        if self.pos == len(self.toks):
            last = self.toks[-1][1] if self.toks else 1
            raise ParseError(self.path, f"truncated input: expected {what}", last)
        word, line = self.toks[self.pos]
        self.pos += 1
        try:
            return float(word)
        except ValueError:
            raise ParseError(self.path, f"expected {what}, got {word!r}", line) from None

    def integer(self, what: str) -> int:
        v = self.number(what)
        if not float(v).is_integer():
            raise ParseError(self.path, f"expected integer {what}, got {v}")
        return int(v)


def _nint(x: float) -> int:
    """TSPLIB nearest-integer rounding of EUC_2D weights."""
    return int(x + 0.5)


def _pairwise_euclid(coords: np.ndarray) -> np.ndarray:
    """Row i = |c_i - c_j| as sqrt(dx*dx + dy*dy), computed one row at a time
    (the reference's expression order)."""
    n = len(coords)
    out = np.empty((n, n))
    for i in range(n):
        dx = coords[i, 0] - coords[:, 0]
        dy = coords[i, 1] - coords[:, 1]
        out[i] = np.sqrt(dx * dx + dy * dy)
    return out


def euclidean_distance_matrix(coords, rounded: bool = False) -> np.ndarray:
    """parsers.py:362-375: nint-rounded and max-symmetrised, or the exact
    matrix averaged with its transpose."""
    coords = np.asarray(coords, dtype=np.float64)
    d = _pairwise_euclid(coords)
    if rounded:
        d = np.array([[_nint(v) for v in row] for row in d], dtype=np.float64).reshape(d.shape)
    np.fill_diagonal(d, 0.0)
    return np.maximum(d, d.T) if rounded else (d + d.T) / 2.0


# ---- TSPLIB ------------------------------------------------------------------

_TSP_SECTIONS = ("NODE_COORD_SECTION", "EDGE_WEIGHT_SECTION")


def parse_tsplib(path) -> InstanceData:
    """parsers.py:70-146: EUC_2D coordinates (nint weights) or EXPLICIT
    FULL_MATRIX / UPPER_ROW weights."""
    lines = _lines_of(path)
    head: dict[str, str] = {}
    section = None
    for no, raw in enumerate(lines, start=1):
        text = raw.strip()
        if not text or text == "EOF":
            continue
        key, _, val = text.partition(":")
        key = key.strip().upper()
        if key in _TSP_SECTIONS:
            section = (key, no)
            break
        if key == "DIMENSION":
            try:
                head["DIMENSION"] = str(int(val.strip()))
            except ValueError:
                raise ParseError(path, f"bad DIMENSION value {val.strip()!r}", no) from None
        elif key in ("EDGE_WEIGHT_TYPE", "EDGE_WEIGHT_FORMAT"):
            head[key] = val.strip().upper()
    if "DIMENSION" not in head:
        raise ParseError(path, "missing DIMENSION header")
    n = int(head["DIMENSION"])
    if n < 2:
        raise ParseError(path, f"DIMENSION must be >= 2, got {n}")
    if section is None:
        raise ParseError(path, "missing coordinate or edge weight section")
    wtype, wfmt = head.get("EDGE_WEIGHT_TYPE"), head.get("EDGE_WEIGHT_FORMAT")
    scan = _Scanner(path, lines, section[1])
    unsupported = f"unsupported EDGE_WEIGHT_TYPE {wtype!r} (supported: EUC_2D, EXPLICIT)"
    if section[0] == "NODE_COORD_SECTION":
        if wtype != "EUC_2D":
            raise ParseError(path, unsupported)
        coords = np.zeros((n, 2))
        for i in range(n):
            scan.integer(f"node id {i + 1}")
            coords[i] = (scan.number("x coordinate"), scan.number("y coordinate"))
        d = _pairwise_euclid(coords)
        d = np.array([[float(_nint(v)) for v in row] for row in d]).reshape(n, n)
        np.fill_diagonal(d, 0.0)
        return InstanceData(distance_matrix=np.maximum(d, d.T),
                            meta={"dimension": n, "coords": coords})
    if wtype != "EXPLICIT":
        raise ParseError(path, unsupported)
    d = np.zeros((n, n))
    if wfmt == "FULL_MATRIX":
        cells = [(i, j) for i in range(n) for j in range(n)]
    elif wfmt == "UPPER_ROW":
        cells = [(i, j) for i in range(n) for j in range(i + 1, n)]
    else:
        raise ParseError(path, f"unsupported EDGE_WEIGHT_FORMAT {wfmt!r} "
                               "(supported: FULL_MATRIX, UPPER_ROW)")
    for i, j in cells:
        d[i, j] = scan.number(f"weight ({i}, {j})")
        if wfmt == "UPPER_ROW":
            d[j, i] = d[i, j]
    if not np.array_equal(d, d.T):
        raise ParseError(path, "explicit matrix is not symmetric")
    if np.any(np.diagonal(d) != 0):
        raise ParseError(path, "explicit matrix has a nonzero diagonal")
    return InstanceData(distance_matrix=d, meta={"dimension": n})


# ---- QAPLIB ------------------------------------------------------------------

def parse_qaplib(path) -> InstanceData:
    """parsers.py:149-162: n, then the n x n flow and distance matrices."""
    scan = _Scanner(path, _lines_of(path))
    n = scan.integer("problem size")
    if n < 2:
        raise ParseError(path, f"problem size must be >= 2, got {n}")
    mats = {}
    for label in ("flow", "distance"):
        m = np.zeros((n, n))
        for i in range(n):
            for j in range(n):
                m[i, j] = scan.number(f"{label} entry ({i}, {j})")
        mats[label] = m
    return InstanceData(flow_matrix=mats["flow"], distance_matrix=mats["distance"],
                        meta={"dimension": n})


# ---- Solomon VRPTW -----------------------------------------------------------

def _numbers_in(lines) -> list[float]:
    vals = []
    for raw in lines:
        for word in raw.split():
            try:
                vals.append(float(word))
            except ValueError:
                pass
    return vals


def parse_solomon(path) -> InstanceData:
    """parsers.py:165-234: VEHICLE block (NUMBER, CAPACITY), CUSTOMER rows of
    (id, x, y, demand, ready, due, service); row id 0 is the depot."""
    lines = _lines_of(path)
    veh_at = cust_at = None
    for idx, raw in enumerate(lines):
        tag = raw.strip().upper()
        if tag.startswith("VEHICLE"):
            veh_at = idx
        elif tag.startswith("CUSTOMER"):
            cust_at = idx
            break
    if veh_at is None or cust_at is None:
        raise ParseError(path, "missing VEHICLE or CUSTOMER section")
    head = _numbers_in(lines[veh_at + 1:cust_at])
    if len(head) < 2:
        raise ParseError(path, "vehicle section needs NUMBER and CAPACITY", veh_at + 1)
    first_row = next((idx for idx in range(cust_at + 1, len(lines))
                      if lines[idx].split() and lines[idx].split()[0].lstrip("+-").isdigit()),
                     None)
    if first_row is None:
        raise ParseError(path, "no customer rows found", cust_at + 1)
    scan = _Scanner(path, lines, first_row)
    recs = []
    while scan.remaining():
        recs.append([scan.number("customer field") for _ in range(7)])
    recs.sort(key=lambda rec: rec[0])
    table = np.array(recs, dtype=np.float64)
    coords = table[:, 1:3].copy()
    d = _pairwise_euclid(coords)
    np.fill_diagonal(d, 0.0)
    return InstanceData(distance_matrix=(d + d.T) / 2.0, demands=table[1:, 3].copy(),
                        capacity=float(head[1]), vehicles=int(head[0]),
                        ready_times=table[:, 4].copy(), due_times=table[:, 5].copy(),
                        service_times=table[:, 6].copy(),
                        meta={"customers": len(recs) - 1, "coords": coords})


# ---- OR-Library job shop -----------------------------------------------------

def parse_orlib_jsp(path) -> InstanceData:
    """parsers.py:237-274: the first line holding exactly two integers gives
    jobs x machines, then (machine, duration) pairs job by job."""
    lines = _lines_of(path)
    start = None
    for idx, raw in enumerate(lines):
        words = raw.split()
        if len(words) == 2 and all(w.lstrip("+-").isdigit() for w in words):
            start, (n_jobs, n_mach) = idx, (int(words[0]), int(words[1]))
            break
    if start is None:
        raise ParseError(path, "missing jobs/machines count line")
    if n_jobs < 1 or n_mach < 1:
        raise ParseError(path, f"bad problem size {n_jobs} x {n_mach}", start + 1)
    scan = _Scanner(path, lines, start + 1)
    jobs = []
    for j in range(n_jobs):
        ops = []
        for k in range(n_mach):
            m = scan.integer(f"machine of job {j} op {k}")
            dur = scan.integer(f"duration of job {j} op {k}")
            if m < 0 or m >= n_mach:
                raise ParseError(path, f"machine {m} outside [0, {n_mach})")
            if dur < 0:
                raise ParseError(path, f"negative duration {dur}")
            ops.append((m, dur))
        jobs.append(ops)
    return InstanceData(jobs=jobs, meta={"jobs": n_jobs, "machines": n_mach})


# ---- JSON payload documents (shared with the scripting bridge) ---------------

def parse_json_instance(path_or_payload) -> tuple[str, InstanceData]:
    """parsers.py:277-297: {"problem": name, ...fields...} from a file or a dict."""
    if isinstance(path_or_payload, dict):
        path, doc = "<inline>", path_or_payload
    else:
        path = path_or_payload
        try:
            doc = json.loads(Path(path).read_text())
        except OSError as exc:
            raise ParseError(path, f"cannot read file ({exc})") from exc
        except json.JSONDecodeError as exc:
            raise ParseError(path, f"invalid JSON: {exc}") from exc
    if not isinstance(doc, dict) or "problem" not in doc:
        raise ParseError(path, 'JSON instance needs a "problem" key')
    name = doc["problem"]
    try:
        return name, payload_to_instance(name, doc)
    except (KeyError, ValueError, TypeError) as exc:
        raise ParseError(path, f"bad payload for problem {name!r}: {exc}") from exc


def _comparison(spec: dict):
    mode = spec.get("mode")
    if mode == "weighted":
        return Weighted(tuple(float(w) for w in spec["weights"]))
    if mode == "lexicographic":
        return Lexicographic(tuple(int(i) for i in spec["priority"]),
                             tuple(float(t) for t in spec["tolerances"]))
    raise ValueError(f"unknown comparison mode {mode!r}")


def _routing_fields(doc, vec):
    return dict(distance_matrix=vec("dist"), demands=vec("demands"),
                capacity=float(doc["capacity"]), vehicles=int(doc["vehicles"]))


def payload_to_instance(name: str, doc: dict) -> InstanceData:
    """parsers.py:300-359: payload field names per problem."""
    def vec(key):
        return np.asarray(doc[key], dtype=np.float64)

    meta: dict = {}
    if "objectives" in doc:
        meta["objectives"] = tuple(doc["objectives"])
    if "comparison" in doc:
        meta["comparison"] = _comparison(doc["comparison"])
    builders = {
        "tsp": lambda: dict(distance_matrix=vec("dist")),
        "cvrp": lambda: _routing_fields(doc, vec),
        "vrp_nonlinear": lambda: _routing_fields(doc, vec),
        "vrp_priority": lambda: dict(_routing_fields(doc, vec), priorities=vec("priorities")),
        "vrptw": lambda: dict(_routing_fields(doc, vec), ready_times=vec("ready"),
                              due_times=vec("due"), service_times=vec("service")),
        "knapsack": lambda: dict(weights=vec("weights"), values=vec("values"),
                                 capacity=float(doc["capacity"])),
        "qap": lambda: dict(flow_matrix=vec("flow"), distance_matrix=vec("dist")),
        "assignment": lambda: dict(cost_matrix=vec("cost")),
        "bin_packing": lambda: dict(item_sizes=vec("sizes"),
                                    bin_capacity=float(doc["bin_capacity"])),
        "load_balancing": lambda: dict(durations=vec("durations"),
                                       num_machines=int(doc["machines"])),
        "jsp_int": lambda: dict(jobs=[[(int(m), int(t)) for m, t in ops] for ops in doc["jobs"]]),
        "schedule_binary": lambda: dict(cost_matrix=vec("cost"),
                                        requirements=vec("requirements")),
    }
    builders["jsp_perm"] = builders["jsp_int"]
    if name == "graph_coloring":
        meta["num_vertices"] = int(doc["vertices"]) if "vertices" in doc else None
        return InstanceData(edges=[(int(u), int(v)) for u, v in doc["edges"]],
                            num_colors=int(doc["colors"]), meta=meta)
    if name not in builders:
        raise ValueError(f"unknown problem {name!r}")
    return InstanceData(meta=meta, **builders[name]())
