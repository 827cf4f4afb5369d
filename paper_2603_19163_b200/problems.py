"""Problem definitions — API mirror of the reference's `problems.py` and
`builtins.py`, backed by the device (no CPU objective path).

`builtin_problem(name, InstanceData)` (builtins.py:42-50) returns a problem
whose configuration matches the reference's exactly (encoding, d1, d2, n, row
mode, objective definitions) and whose objective / penalty are evaluated by
`libcugenopt.so` (go_eval_batch).  Python `compute_objective` callbacks of
user subclasses cannot run on the device: the engine rejects them loudly.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .core import (ComparisonMode, Direction, Encoding, ObjDef, ProblemConfig, RowModeKind,
                   Solution, validate_solution)
from .operators import (SEQ_FLIP, SEQ_INSERT, SEQ_OR_OPT, SEQ_RANDOM_RESET, SEQ_REVERSE,
                        SEQ_ROW_MERGE, SEQ_ROW_SPLIT, SEQ_ROW_SWAP, SEQ_SCATTER_SHUFFLE,
                        SEQ_SEG_FLIP, SEQ_SEG_RESET, SEQ_SEG_SHUFFLE, SEQ_SWAP, SEQ_THREE_OPT,
                        SEQ_OX_CROSSOVER, SEQ_UNIFORM_CROSSOVER, SEQ_GUIDED_REBUILD)

BUILTIN_NAMES = ("tsp", "cvrp", "vrptw", "knapsack", "qap", "assignment", "graph_coloring",
                 "bin_packing", "load_balancing", "jsp_int", "jsp_perm", "schedule_binary",
                 "vrp_priority", "vrp_nonlinear")
DEVICE_PROBLEMS = ("tsp", "qap", "knapsack", "jsp_int", "vrptw", "cvrp", "assignment",
                   "graph_coloring", "bin_packing", "load_balancing", "vrp_priority",
                   "vrp_nonlinear", "jsp_perm", "schedule_binary")


@dataclass
class InstanceData:
    """problems.py:18-46 — numeric payload of one instance."""

    distance_matrix: np.ndarray | None = None
    weights: np.ndarray | None = None
    values: np.ndarray | None = None
    capacity: float | None = None
    flow_matrix: np.ndarray | None = None
    cost_matrix: np.ndarray | None = None
    edges: list | None = None
    num_colors: int | None = None
    item_sizes: np.ndarray | None = None
    bin_capacity: float | None = None
    durations: np.ndarray | None = None
    num_machines: int | None = None
    jobs: list | None = None
    demands: np.ndarray | None = None
    vehicles: int | None = None
    ready_times: np.ndarray | None = None
    due_times: np.ndarray | None = None
    service_times: np.ndarray | None = None
    priorities: np.ndarray | None = None
    requirements: np.ndarray | None = None
    meta: dict = field(default_factory=dict)


class ProblemDefinition:
    """problems.py:49-74.  Device-backed problems implement `_native_desc`."""

    def config(self) -> ProblemConfig:
        raise NotImplementedError

    def compute_objective(self, i: int, sol: Solution) -> float:
        obj, _ = device_evaluate(self, [sol])
        return float(obj[0, i])

    def compute_penalty(self, sol: Solution) -> float:
        _, pen = device_evaluate(self, [sol])
        return float(pen[0])

    def init_matrices(self) -> list[np.ndarray]:
        return []

    def init_candidates(self, rng) -> list[Solution] | None:
        return None

    def payload_nbytes(self) -> int:
        return sum(m.nbytes for m in self.init_matrices())

    # -- device plumbing -------------------------------------------------------
    # one native problem handle per device (replicas may run on several GPUs)
    _handles = None
    #: built-in sequence ids the device kernel for this problem implements
    DEVICE_SEQUENCES: tuple = ()

    def device_sequences(self) -> tuple:
        return self.DEVICE_SEQUENCES

    def _native_desc(self):
        raise TypeError(
            f"{type(self).__name__} has no device objective: the B200 engine evaluates "
            "built-in problems (and NVRTC objectives) only; Python callbacks are not a "
            "supported path")

    def _cached_handle(self, device: int):
        if self._handles is None:
            self._handles = {}
        return self._handles.get(device)

    def _store_handle(self, device: int, h, keep):
        self._handles[device] = h
        self._keepalive = getattr(self, "_keepalive", {})
        self._keepalive[device] = keep

    def device_handle(self, device: int = 0):
        h = self._cached_handle(device)
        if h is not None:
            return h
        lib = N.load()
        desc, keep = self._native_desc()
        h = C.c_void_p()
        N.check(lib.go_problem_create(C.byref(desc), device, C.byref(h)))
        self._store_handle(device, h, keep)
        return h

    def __del__(self):
        for h in (getattr(self, "_handles", None) or {}).values():
            if N._lib is not None:
                try:
                    N._lib.go_problem_destroy(h)
                except Exception:  # noqa: BLE001
                    pass


def check_distance_matrix(d, symmetric: bool = True) -> np.ndarray:
    """problems.py:97-107."""
    d = np.asarray(d, dtype=np.float64)
    if d.ndim != 2 or d.shape[0] != d.shape[1]:
        raise ValueError(f"distance matrix must be square, got shape {d.shape}")
    if np.any(d < 0):
        raise ValueError("distance matrix must be nonnegative")
    if np.any(np.diag(d) != 0):
        raise ValueError("distance matrix must have a zero diagonal")
    if symmetric and not np.array_equal(d, d.T):
        raise ValueError("distance matrix declared symmetric but is not")
    return d


def pack_solutions(sols, cfg: ProblemConfig):
    """Solutions -> (genes[m][d1*d2] int32, sizes[m][d1] int32) for the C ABI."""
    m = len(sols)
    genes = np.zeros((m, cfg.d1 * cfg.d2), dtype=np.int32)
    sizes = np.zeros((m, cfg.d1), dtype=np.int32)
    for i, s in enumerate(sols):
        genes[i] = s.data.reshape(-1)
        sizes[i] = s.dim2_sizes
    return genes, sizes


def device_evaluate(problem: ProblemDefinition, sols, device: int = 0):
    """Batch evaluate() on the device: objectives [m, 1], penalties [m]."""
    cfg = problem.config()
    lib = N.load()
    h = problem.device_handle(device)
    genes, sizes = pack_solutions(sols, cfg)
    m = cfg.num_objectives
    obj = np.zeros(len(sols) * m, dtype=np.float64)
    pen = np.zeros(len(sols), dtype=np.float64)
    N.check(lib.go_eval_batch(h, N.iptr(genes), N.iptr(sizes), len(sols), N.dptr(obj),
                              N.dptr(pen)))
    return obj.reshape(-1, m), pen


def evaluate(problem: ProblemDefinition, sol: Solution, *, validate: bool = True):
    """problems.py:77-94, evaluated on the device."""
    cfg = problem.config()
    if validate:
        report = validate_solution(sol, cfg)
        if not report.ok:
            raise ValueError(f"refusing to evaluate invalid solution: {report.violations[:3]}")
    obj, pen = device_evaluate(problem, [sol])
    sol.objectives[:] = obj[0]
    sol.penalty = float(pen[0])
    if sol.penalty < 0:
        raise ValueError(f"penalty must be nonnegative, got {sol.penalty}")
    return sol.objectives, sol.penalty


def evaluate_many(problem: ProblemDefinition, sols, device: int = 0):
    """Evaluate a list of solutions in one device call (used by initialisation)."""
    if not sols:
        return
    obj, pen = device_evaluate(problem, sols, device)
    for s, o, p in zip(sols, obj, pen):
        s.objectives[:] = o
        s.penalty = float(p)


class TspProblem(ProblemDefinition):
    """builtins.py:53-77: cyclic tour length over a symmetric matrix."""

    DEVICE_SEQUENCES = (SEQ_SWAP, SEQ_INSERT, SEQ_REVERSE, SEQ_OR_OPT, SEQ_THREE_OPT,
                        SEQ_OX_CROSSOVER, SEQ_SEG_SHUFFLE, SEQ_SCATTER_SHUFFLE, SEQ_GUIDED_REBUILD)

    def __init__(self, dist):
        self.dist = check_distance_matrix(dist)
        self.n = self.dist.shape[0]
        self._cfg = ProblemConfig(encoding=Encoding.permutation(), d1=1, d2=self.n, n=self.n,
                                  row_mode=RowModeKind.SINGLE_SEQ,
                                  obj_defs=(ObjDef("tour_length"),))

    def config(self):
        return self._cfg

    def compute_penalty(self, sol):
        return 0.0

    def init_matrices(self):
        return [self.dist]

    def _native_desc(self):
        d = N.f64(self.dist)
        desc = N.ProblemDesc(kind=N.GO_TSP, n=self.n, d1=1, d2=self.n)
        desc.dist = N.dptr(d)
        return desc, (d,)


class QapProblem(ProblemDefinition):
    """builtins.py:265-290: Σ_ij F_ij D[π_i, π_j] (matrices not symmetry-checked)."""

    DEVICE_SEQUENCES = (SEQ_SWAP, SEQ_INSERT, SEQ_REVERSE, SEQ_OR_OPT, SEQ_THREE_OPT,
                        SEQ_OX_CROSSOVER, SEQ_SEG_SHUFFLE, SEQ_SCATTER_SHUFFLE, SEQ_GUIDED_REBUILD)

    def __init__(self, flow, dist):
        self.flow = np.asarray(flow, dtype=np.float64)
        self.dist = np.asarray(dist, dtype=np.float64)
        if self.flow.shape != self.dist.shape or self.flow.ndim != 2 or \
                self.flow.shape[0] != self.flow.shape[1]:
            raise ValueError("flow and distance matrices must be square and equal-shaped")
        self.n = self.flow.shape[0]
        self._cfg = ProblemConfig(encoding=Encoding.permutation(), d1=1, d2=self.n, n=self.n,
                                  row_mode=RowModeKind.SINGLE_SEQ,
                                  obj_defs=(ObjDef("total_cost"),))

    def config(self):
        return self._cfg

    def compute_penalty(self, sol):
        return 0.0

    def init_matrices(self):
        return [self.flow, self.dist]

    def _native_desc(self):
        f, d = N.f64(self.flow), N.f64(self.dist)
        desc = N.ProblemDesc(kind=N.GO_QAP, n=self.n, d1=1, d2=self.n)
        desc.flow, desc.dist = N.dptr(f), N.dptr(d)
        return desc, (f, d)


class KnapsackProblem(ProblemDefinition):
    """builtins.py:240-262: maximise v·x, penalty max(0, w·x - capacity)."""

    DEVICE_SEQUENCES = (SEQ_FLIP, SEQ_SEG_FLIP, SEQ_UNIFORM_CROSSOVER, SEQ_SEG_SHUFFLE,
                        SEQ_SCATTER_SHUFFLE, SEQ_GUIDED_REBUILD)

    def __init__(self, weights, values, capacity):
        self.weights = np.asarray(weights, dtype=np.float64)
        self.values = np.asarray(values, dtype=np.float64)
        self.capacity = float(capacity)
        if len(self.weights) != len(self.values):
            raise ValueError("weights and values must have equal length")
        self.n = len(self.weights)
        self._cfg = ProblemConfig(encoding=Encoding.binary(), d1=1, d2=self.n, n=self.n,
                                  row_mode=RowModeKind.SINGLE_SEQ,
                                  obj_defs=(ObjDef("total_value", Direction.MAXIMIZE),))

    def config(self):
        return self._cfg

    def _native_desc(self):
        w, v = N.f64(self.weights), N.f64(self.values)
        desc = N.ProblemDesc(kind=N.GO_KNAPSACK, n=self.n, d1=1, d2=self.n,
                             capacity=self.capacity)
        desc.weights, desc.values = N.dptr(w), N.dptr(v)
        return desc, (w, v)


class JspIntProblem(ProblemDefinition):
    """builtins.py:408-456: priority-decoded serial schedule generator."""

    DEVICE_SEQUENCES = (SEQ_RANDOM_RESET, SEQ_SEG_RESET, SEQ_UNIFORM_CROSSOVER, SEQ_SEG_SHUFFLE,
                        SEQ_SCATTER_SHUFFLE, SEQ_GUIDED_REBUILD)

    def __init__(self, jobs):
        self.jobs = [[(int(m), int(d)) for m, d in ops] for ops in jobs]
        if not self.jobs:
            raise ValueError("at least one job required")
        self.ops_per_job = len(self.jobs[0])
        for j, ops in enumerate(self.jobs):
            if len(ops) != self.ops_per_job:
                raise ValueError(f"job {j} has {len(ops)} operations, expected {self.ops_per_job}")
        self.n_jobs = len(self.jobs)
        self.n_machines = 1 + max(m for ops in self.jobs for m, _ in ops)
        self.n_ops = self.n_jobs * self.ops_per_job
        self._cfg = ProblemConfig(encoding=Encoding.integer(0, self.n_ops - 1), d1=1,
                                  d2=self.n_ops, n=self.n_ops, row_mode=RowModeKind.SINGLE_SEQ,
                                  obj_defs=(ObjDef("makespan"),))

    def config(self):
        return self._cfg

    def compute_penalty(self, sol):
        return 0.0

    def _native_desc(self):
        mach = np.array([m for ops in self.jobs for m, _ in ops], dtype=np.int32)
        dur = np.array([d for ops in self.jobs for _, d in ops], dtype=np.int32)
        desc = N.ProblemDesc(kind=N.GO_JSP_INT, n=self.n_ops, d1=1, d2=self.n_ops,
                             n_jobs=self.n_jobs, n_machines=self.n_machines,
                             ops_per_job=self.ops_per_job, lb=0, ub=self.n_ops - 1)
        desc.jsp_machine, desc.jsp_duration = N.iptr(mach), N.iptr(dur)
        return desc, (mach, dur)


class RoutingProblem(ProblemDefinition):
    """builtins.py:80-152 (CVRP): Σ route lengths, penalty Σ max(0, load - cap).
    Customers are values 0..n-1 at matrix index c + 1 (index 0 = depot)."""

    DEVICE_SEQUENCES = (SEQ_SWAP, SEQ_INSERT, SEQ_REVERSE, SEQ_OR_OPT, SEQ_THREE_OPT,
                        SEQ_ROW_SWAP, SEQ_ROW_SPLIT, SEQ_ROW_MERGE, SEQ_OX_CROSSOVER,
                        SEQ_SEG_SHUFFLE, SEQ_SCATTER_SHUFFLE, SEQ_GUIDED_REBUILD)
    _KIND = N.GO_CVRP

    def __init__(self, dist, demands, capacity, vehicles, objectives=("distance",),
                 comparison=None):
        self.dist = check_distance_matrix(dist)
        self.demands = np.asarray(demands, dtype=np.float64)
        self.capacity = float(capacity)
        self.vehicles = int(vehicles)
        self.n = len(self.demands)
        if self.dist.shape[0] != self.n + 1:
            raise ValueError(f"distance matrix has {self.dist.shape[0]} nodes, expected "
                             f"{self.n + 1} (depot + {self.n} customers)")
        if self.vehicles < 1:
            raise ValueError("at least one vehicle required")
        self.objective_names = tuple(objectives)
        for name in self.objective_names:
            if name not in ("distance", "vehicles"):
                raise ValueError(f"unknown routing objective {name!r}")
        self._cfg = ProblemConfig(encoding=Encoding.permutation(), d1=self.vehicles, d2=self.n,
                                  n=self.n, row_mode=RowModeKind.MULTI_PARTITION,
                                  obj_defs=tuple(ObjDef(nm) for nm in self.objective_names),
                                  comparison=comparison)

    def config(self):
        return self._cfg

    def init_matrices(self):
        return [self.dist[1:, 1:]]

    def payload_nbytes(self):
        return self.dist.nbytes + self.demands.nbytes

    def _arrays(self):
        n1 = self.n + 1
        z = np.zeros(n1)
        return z, z, z

    def _native_desc(self):
        d, dem = N.f64(self.dist), N.f64(self.demands)
        ready, due, service = (N.f64(a) for a in self._arrays())
        kinds = [1 if name == "vehicles" else 0 for name in self.objective_names] + [1]
        desc = N.ProblemDesc(kind=self._KIND, n=self.n, d1=self.vehicles, d2=self.n,
                             capacity=self.capacity, n_obj=len(self.objective_names))
        desc.obj_kind[0], desc.obj_kind[1] = kinds[0], kinds[1]
        desc.dist, desc.demands = N.dptr(d), N.dptr(dem)
        desc.ready, desc.due, desc.service = N.dptr(ready), N.dptr(due), N.dptr(service)
        return desc, (d, dem, ready, due, service)


class VrptwProblem(RoutingProblem):
    """builtins.py:155-190: CVRP + sequential lateness (arrival = max(ready, t + d))."""

    _KIND = N.GO_VRPTW

    def __init__(self, dist, demands, capacity, vehicles, ready, due, service,
                 objectives=("distance",), comparison=None):
        super().__init__(dist, demands, capacity, vehicles, objectives=objectives,
                         comparison=comparison)
        self.ready = np.asarray(ready, dtype=np.float64)
        self.due = np.asarray(due, dtype=np.float64)
        self.service = np.asarray(service, dtype=np.float64)
        for arr, label in ((self.ready, "ready"), (self.due, "due"), (self.service, "service")):
            if len(arr) != self.n + 1:
                raise ValueError(f"{label} times must cover depot + {self.n} customers")

    def _arrays(self):
        return self.ready, self.due, self.service

    def payload_nbytes(self):
        return super().payload_nbytes() + self.ready.nbytes + self.due.nbytes + \
            self.service.nbytes


class PriorityVrpProblem(RoutingProblem):
    """builtins.py:193-210: CVRP whose penalty adds, per route, the number of
    (earlier, later) customer pairs where the later one has higher priority."""

    _KIND = N.GO_VRP_PRIORITY

    def __init__(self, dist, demands, capacity, vehicles, priorities, objectives=("distance",),
                 comparison=None):
        super().__init__(dist, demands, capacity, vehicles, objectives=objectives,
                         comparison=comparison)
        self.priorities = np.asarray(priorities, dtype=np.float64)
        if len(self.priorities) != self.n:
            raise ValueError("one priority per customer required")

    def _native_desc(self):
        desc, keep = super()._native_desc()
        pr = N.f64(self.priorities)
        desc.priorities = N.dptr(pr)
        return desc, keep + (pr,)


class NonlinearVrpProblem(RoutingProblem):
    """builtins.py:213-237: edge cost d_ij * (1 + 0.3 (load / cap)^2), the load
    being the demand collected before the edge."""

    _KIND = N.GO_VRP_NONLINEAR


def _routing_kwargs(instance: InstanceData) -> dict:
    kwargs = {}
    meta = instance.meta or {}
    if "objectives" in meta:
        kwargs["objectives"] = tuple(meta["objectives"])
    if "comparison" in meta:
        kwargs["comparison"] = meta["comparison"]
    return kwargs


def _need(instance: InstanceData, *names):
    missing = [f for f in names if getattr(instance, f) is None]
    if missing:
        raise ValueError(f"instance payload missing fields: {', '.join(missing)}")


def builtin_problem(name: str, instance: InstanceData) -> ProblemDefinition:
    """builtins.py:42-50."""
    if name not in BUILTIN_NAMES:
        raise ValueError(f"unknown problem {name!r}; known problems: {', '.join(BUILTIN_NAMES)}")
    if name == "tsp":
        _need(instance, "distance_matrix")
        return TspProblem(instance.distance_matrix)
    if name == "qap":
        _need(instance, "flow_matrix", "distance_matrix")
        return QapProblem(instance.flow_matrix, instance.distance_matrix)
    if name == "knapsack":
        _need(instance, "weights", "values", "capacity")
        return KnapsackProblem(instance.weights, instance.values, instance.capacity)
    if name == "jsp_int":
        _need(instance, "jobs")
        return JspIntProblem(instance.jobs)
    if name == "cvrp":
        _need(instance, "distance_matrix", "demands", "capacity", "vehicles")
        return RoutingProblem(instance.distance_matrix, instance.demands, instance.capacity,
                              instance.vehicles, **_routing_kwargs(instance))
    if name == "vrptw":
        _need(instance, "distance_matrix", "demands", "capacity", "vehicles", "ready_times",
              "due_times", "service_times")
        return VrptwProblem(instance.distance_matrix, instance.demands, instance.capacity,
                            instance.vehicles, instance.ready_times, instance.due_times,
                            instance.service_times, **_routing_kwargs(instance))
    if name == "vrp_priority":
        _need(instance, "distance_matrix", "demands", "capacity", "vehicles", "priorities")
        return PriorityVrpProblem(instance.distance_matrix, instance.demands, instance.capacity,
                                  instance.vehicles, instance.priorities,
                                  **_routing_kwargs(instance))
    if name == "vrp_nonlinear":
        _need(instance, "distance_matrix", "demands", "capacity", "vehicles")
        return NonlinearVrpProblem(instance.distance_matrix, instance.demands, instance.capacity,
                                   instance.vehicles, **_routing_kwargs(instance))
    if name == "assignment":
        _need(instance, "cost_matrix")
        return AssignmentProblem(instance.cost_matrix)
    if name == "graph_coloring":
        _need(instance, "edges", "num_colors")
        n = instance.meta.get("num_vertices")
        if n is None:
            n = 1 + max(max(u, v) for u, v in instance.edges)
        return GraphColoringProblem(n, instance.edges, instance.num_colors)
    if name == "bin_packing":
        _need(instance, "item_sizes", "bin_capacity")
        return BinPackingProblem(instance.item_sizes, instance.bin_capacity)
    if name == "load_balancing":
        _need(instance, "durations", "num_machines")
        return LoadBalancingProblem(instance.durations, instance.num_machines)
    if name == "jsp_perm":
        _need(instance, "jobs")
        return JspPermProblem(instance.jobs)
    if name == "schedule_binary":
        _need(instance, "cost_matrix", "requirements")
        return BinaryScheduleProblem(instance.cost_matrix, instance.requirements)
    raise NotImplementedError(
        f"problem {name!r} has no B200 device path in this build "
        f"(device problems: {', '.join(DEVICE_PROBLEMS)})")


class CudaProblem(ProblemDefinition):
    """A user-defined single-row problem whose objective and penalty are CUDA
    snippets, compiled by NVRTC for sm_100a into the row evolve kernel (the
    paper's `solve_custom`).  It stands in for a reference
    `ProblemDefinition` subclass (problems.py:49-74): the reference's Python
    `compute_objective` / `compute_penalty` callbacks become the bodies of

        template <class Sol> double compute_obj(const Sol& sol, const Data& data)
        template <class Sol> double compute_penalty(const Sol& sol, const Data& data)

    reading genes as `sol[i]` (0 <= i < sol.n) and every entry of `data` as
    `data.<name>` (const double*, length `data.<name>_len`).  All built-in
    operators applicable to the encoding run on the device, including
    crossovers and guided rebuild (whose trials call the snippet)."""

    JIT = True  # device_handle compiles (reported as jit_seconds, outside the budget)
    _ENC = {"permutation": N.ENC_PERM, "binary": N.ENC_BINARY, "integer": N.ENC_INTEGER}
    _SEQS = {
        "permutation": (SEQ_SWAP, SEQ_INSERT, SEQ_REVERSE, SEQ_OR_OPT, SEQ_THREE_OPT,
                        SEQ_OX_CROSSOVER, SEQ_SEG_SHUFFLE, SEQ_SCATTER_SHUFFLE,
                        SEQ_GUIDED_REBUILD),
        "binary": (SEQ_FLIP, SEQ_SEG_FLIP, SEQ_UNIFORM_CROSSOVER, SEQ_SEG_SHUFFLE,
                   SEQ_SCATTER_SHUFFLE, SEQ_GUIDED_REBUILD),
        "integer": (SEQ_RANDOM_RESET, SEQ_SEG_RESET, SEQ_UNIFORM_CROSSOVER, SEQ_SEG_SHUFFLE,
                    SEQ_SCATTER_SHUFFLE, SEQ_GUIDED_REBUILD),
    }

    def __init__(self, encoding: str, n: int, compute_obj, compute_penalty: str | None = None,
                 data: dict | None = None, lb: int = 0, ub: int | None = None,
                 maximize=False, name="objective", init_matrices: list | None = None,
                 rows: int = 1, comparison=None, weights=None):
        if encoding not in self._ENC:
            raise ValueError(f"encoding must be one of {sorted(self._ENC)}, got {encoding!r}")
        # one objective, or two (compute_obj = [obj0, obj1]; maximize / name / weights
        # per objective; comparison Weighted or Lexicographic, core.py:80-106)
        objs = [compute_obj] if isinstance(compute_obj, str) else list(compute_obj)
        if not 1 <= len(objs) <= 2 or any(not isinstance(o, str) or not o.strip() for o in objs):
            raise ValueError("compute_obj must be one CUDA snippet (function body) or two")
        m = len(objs)
        maxes = [maximize] * m if isinstance(maximize, bool) else list(maximize)
        names = [name] * m if isinstance(name, str) else list(name)
        if m == 2 and isinstance(name, str):
            names = [f"{name}0", f"{name}1"]
        ws = list(weights) if weights is not None else [1.0] * m
        if not (len(maxes) == len(names) == len(ws) == m):
            raise ValueError("maximize / name / weights need one entry per objective")
        compute_obj = objs[0]
        self.compute_obj2_src = objs[1] if m == 2 else None
        self.encoding, self.n, self.rows = encoding, int(n), int(rows)
        if self.rows < 1:
            raise ValueError("rows must be >= 1")
        self.compute_obj_src, self.compute_penalty_src = compute_obj, compute_penalty
        self.data = {k: np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
                     for k, v in (data or {}).items()}
        if encoding == "permutation":
            enc = Encoding.permutation()
        elif encoding == "binary":
            enc = Encoding.binary()
        else:
            if ub is None:
                raise ValueError("integer encoding needs ub")
            enc = Encoding.integer(int(lb), int(ub))
        self.lb, self.ub = (int(lb), int(ub)) if encoding == "integer" else (0, 0)
        self._matrices = [np.asarray(m, dtype=np.float64) for m in (init_matrices or [])]
        # rows > 1: MULTI_FIXED (core.py:28-35) — every row holds n genes (a full
        # permutation of range(n) for the permutation encoding); snippets read
        # row r, column i as sol[r * n + i]
        self._cfg = ProblemConfig(
            encoding=enc, d1=self.rows, d2=self.n,
            n=self.n if encoding == "permutation" else self.rows * self.n,
            row_mode=RowModeKind.SINGLE_SEQ if self.rows == 1 else RowModeKind.MULTI_FIXED,
            obj_defs=tuple(ObjDef(nm, Direction.MAXIMIZE if mx else Direction.MINIMIZE, w)
                           for nm, mx, w in zip(names, maxes, ws)),
            comparison=comparison)

    def config(self):
        return self._cfg

    def init_matrices(self):
        return self._matrices

    def payload_nbytes(self) -> int:
        return sum(a.nbytes for a in self.data.values())

    def device_sequences(self):
        return self._SEQS[self.encoding]

    def device_handle(self, device: int = 0):
        h = self._cached_handle(device)
        if h is not None:
            return h
        lib = N.load()
        names = list(self.data)
        arrays = [self.data[k] for k in names]
        c_names = (C.c_char_p * max(1, len(names)))(*[k.encode() for k in names])
        c_ptrs = (C.POINTER(C.c_double) * max(1, len(names)))(*[N.dptr(a) for a in arrays])
        c_lens = (C.c_int64 * max(1, len(names)))(*[len(a) for a in arrays])
        desc = N.UserProblemDesc(
            encoding=self._ENC[self.encoding], n=self.n, lb=self.lb, ub=self.ub,
            compute_obj=self.compute_obj_src.encode(),
            compute_penalty=self.compute_penalty_src.encode() if self.compute_penalty_src else None,
            n_data=len(names), data_names=c_names, data=c_ptrs, data_lens=c_lens,
            rows=self.rows,
            compute_obj2=self.compute_obj2_src.encode() if self.compute_obj2_src else None)
        h = C.c_void_p()
        log = C.create_string_buffer(8192)
        N.check(lib.go_problem_create_user(C.byref(desc), device, C.byref(h), log, len(log)))
        self._store_handle(device, h, (arrays, c_names, c_ptrs, c_lens))
        return h


# ---- further reference built-ins as NVRTC objectives (builtins.py:293-394) ------------
# Each snippet restates the reference objective with its arithmetic order
# (numpy pairwise sums where the reference sums an array, sequential per-bin
# accumulation where it uses np.bincount), so integer-valued instances match
# bit-for-bit and float instances within rounding of the same operation order.

_PAIRWISE_COST = """
  struct F {
    const double* c; const Sol* s; int n;
    __device__ double operator()(int i) const { return c[i * n + (*s)[i]]; }
  } f{data.cost, &sol, sol.n};
  return go::np_pairwise(f, 0, sol.n);
"""

_COLOR_CONFLICTS = """
  int k = 0;
  for (int e = 0; e < data.eu_len; ++e) k += sol[(int)data.eu[e]] == sol[(int)data.ev[e]];
  return (double)k;
"""

_BINS_USED = """
  int used = 0;  // len(np.unique(row))
  for (int b = 0; b < sol.n; ++b) {
    bool any = false;
    for (int i = 0; i < sol.n && !any; ++i) any = sol[i] == b;
    used += any;
  }
  return (double)used;
"""
_BIN_OVERFLOW = """
  struct F {  // max(bincount(row, sizes)[b] - cap, 0), bins summed pairwise
    const double* w; const Sol* s; double cap;
    __device__ double operator()(int b) const {
      double load = 0.0;
      for (int i = 0; i < s->n; ++i) if ((*s)[i] == b) load = __dadd_rn(load, w[i]);
      const double o = __dsub_rn(load, cap);
      return o > 0.0 ? o : 0.0;
    }
  } f{data.sizes, &sol, data.cap[0]};
  return go::np_pairwise(f, 0, sol.n);
"""

_MAKESPAN_LOADS = """
  double mx = 0.0;  // bincount(row, durations, minlength=M).max()
  for (int m = 0; m < (int)data.machines[0]; ++m) {
    double load = 0.0;
    for (int i = 0; i < sol.n; ++i) if (sol[i] == m) load = __dadd_rn(load, data.dur[i]);
    mx = (m == 0 || load > mx) ? load : mx;
  }
  return mx;
"""


_JSPP_DECODE = """
  constexpr int MAXJ = 64;  // JspPermProblem._decode (builtins.py:480-508)
  const int nj = (int)data.dims[0], pj = (int)data.dims[1], nm = (int)data.dims[2];
  int ptr[MAXJ], nxt[MAXJ];
  double ja[MAXJ], ma[MAXJ];
  for (int i = 0; i < nm; ++i) { ptr[i] = 0; ma[i] = 0.0; }
  for (int j = 0; j < nj; ++j) { nxt[j] = 0; ja[j] = 0.0; }
  const int total = nj * pj;
  int done = 0;
  double span = 0.0;
  bool moved = true;
  while (moved && done < total) {
    moved = false;
    for (int m = 0; m < nm; ++m) {  // one sweep over the machines' head jobs
      if (ptr[m] >= nj) continue;
      const int j = sol[m * nj + ptr[m]];
      const int k = nxt[j];
      if (k >= pj || (int)data.mach[j * pj + k] != m) continue;
      const double end = __dadd_rn(ja[j] > ma[m] ? ja[j] : ma[m], data.dur[j * pj + k]);
      ja[j] = end;
      ma[m] = end;
      ++nxt[j];
      ++ptr[m];
      ++done;
      span = end > span ? end : span;
      moved = true;
    }
  }
"""

_SCHED_COST = """
  struct F {  // (cost * data).sum(): numpy pairwise over the d1 x d2 cells
    const double* c; const Sol* s;
    __device__ double operator()(int i) const { return __dmul_rn(c[i], (double)(*s)[i]); }
  } f{data.cost, &sol};
  return go::np_pairwise(f, 0, sol.n);
"""
_SCHED_UNCOVERED = """
  struct F {  // max(requirements - data.sum(axis=0), 0).sum()
    const double* req; const Sol* s; int d1, d2;
    __device__ double operator()(int sh) const {
      long long cov = 0;
      for (int r = 0; r < d1; ++r) cov += (*s)[r * d2 + sh];
      const double u = __dsub_rn(req[sh], (double)cov);
      return u > 0.0 ? u : 0.0;
    }
  } f{data.req, &sol, (int)data.dims[0], (int)data.dims[1]};
  return go::np_pairwise(f, 0, (int)data.dims[1]);
"""


class JspPermProblem(CudaProblem):
    """builtins.py:459-516: MULTI_FIXED permutation rows, row m = the job order
    on machine m; makespan of the sweep decoder, penalty = operations left
    unscheduled by a cyclic wait."""

    def __init__(self, jobs):
        jobs = [[(int(m), int(d)) for m, d in ops] for ops in jobs]
        if not jobs or any(len(ops) != len(jobs[0]) for ops in jobs) or not jobs[0]:
            raise ValueError("every job needs the same, nonzero number of operations")
        nj, pj = len(jobs), len(jobs[0])
        nm = 1 + max(m for ops in jobs for m, _ in ops)
        if nj > 64 or nm > 64:
            raise ValueError("jsp_perm on the device supports up to 64 jobs and 64 machines")
        self.jobs = jobs
        data = {"mach": [m for ops in jobs for m, _ in ops],
                "dur": [d for ops in jobs for _, d in ops], "dims": [nj, pj, nm]}
        super().__init__("permutation", nj, _JSPP_DECODE + "  return span;\n",
                         _JSPP_DECODE + "  return (double)(total - done);\n", data=data,
                         name="makespan", rows=nm)


class BinaryScheduleProblem(CudaProblem):
    """builtins.py:519-545: worker x shift 0/1 MULTI_FIXED rows; cost sum,
    penalty = uncovered requirement summed over shifts."""

    def __init__(self, cost, requirements):
        cost = np.asarray(cost, dtype=np.float64)
        if cost.ndim != 2:
            raise ValueError("cost must be a worker x shift matrix")
        req = np.asarray(requirements, dtype=np.float64)
        if len(req) != cost.shape[1]:
            raise ValueError("one coverage requirement per shift required")
        w, sh = cost.shape
        super().__init__("binary", sh, _SCHED_COST, _SCHED_UNCOVERED,
                         data={"cost": cost, "req": req, "dims": [w, sh]}, name="total_cost",
                         rows=w)


class AssignmentProblem(CudaProblem):
    """builtins.py:293-319: Σ_i cost[i, perm[i]] (numpy pairwise)."""

    def __init__(self, cost):
        cost = np.asarray(cost, dtype=np.float64)
        if cost.ndim != 2 or cost.shape[0] != cost.shape[1]:
            raise ValueError("assignment cost matrix must be square")
        super().__init__("permutation", cost.shape[0], _PAIRWISE_COST, data={"cost": cost},
                         name="total_cost", init_matrices=[cost])


class GraphColoringProblem(CudaProblem):
    """builtins.py:322-350: monochromatic edges under a fixed palette."""

    def __init__(self, num_vertices, edges, num_colors):
        n = int(num_vertices)
        edges = [(int(u), int(v)) for u, v in edges]
        for u, v in edges:
            if not (0 <= u < n and 0 <= v < n):
                raise ValueError(f"edge ({u}, {v}) outside vertex range")
        self.edges = edges
        super().__init__("integer", n, _COLOR_CONFLICTS,
                         data={"eu": [u for u, _ in edges] or [0.0],
                               "ev": [v for _, v in edges] or [0.0]},
                         lb=0, ub=int(num_colors) - 1, name="conflicts")
        if not edges:  # no edges: zero conflicts
            self.compute_obj_src = "return 0.0;"


class BinPackingProblem(CudaProblem):
    """builtins.py:353-373: bins used; penalty = Σ max(load - capacity, 0)."""

    def __init__(self, item_sizes, bin_capacity):
        sizes = np.asarray(item_sizes, dtype=np.float64)
        n = len(sizes)
        super().__init__("integer", n, _BINS_USED, _BIN_OVERFLOW,
                         data={"sizes": sizes, "cap": [float(bin_capacity)]},
                         lb=0, ub=n - 1, name="bins_used")


class LoadBalancingProblem(CudaProblem):
    """builtins.py:376-394: makespan of bincount(assignment, durations)."""

    def __init__(self, durations, num_machines):
        d = np.asarray(durations, dtype=np.float64)
        m = int(num_machines)
        super().__init__("integer", len(d), _MAKESPAN_LOADS,
                         data={"dur": d, "machines": [float(m)]}, lb=0, ub=m - 1,
                         name="makespan")
