"""Objective / penalty restatements (test infrastructure only).

Each class restates one reference problem from
`/root/reference/pkg/src/genopt/builtins.py` with numpy arithmetic in the same
order as the reference, so float64 results are bit-identical to it.  The
`Sol` container restates `core.Solution` (core.py:154-200): a d1 x d2 int64
matrix, per-row effective lengths, objectives and penalty.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

PERM, BINARY, INTEGER = "permutation", "binary", "integer"
SINGLE, MULTI_FIXED, PARTITION = "single_seq", "multi_fixed", "multi_partition"
MIN, MAX = "minimize", "maximize"


class Sol:
    """core.py:154-200 — row-organised integer solution."""

    __slots__ = ("data", "sizes", "obj", "pen")

    def __init__(self, data, sizes, m: int = 1):
        self.data = np.asarray(data, dtype=np.int64)
        self.sizes = np.asarray(sizes, dtype=np.int64)
        self.obj = np.full(m, np.nan)
        self.pen = 0.0

    @property
    def d1(self):
        return self.data.shape[0]

    @property
    def d2(self):
        return self.data.shape[1]

    def row(self, r):
        return self.data[r, : self.sizes[r]]

    def flat(self):
        return np.concatenate([self.row(r) for r in range(self.d1)]) \
            if self.d1 > 1 else self.row(0).copy()

    def clone(self):
        out = Sol.__new__(Sol)
        out.data = self.data.copy()
        out.sizes = self.sizes.copy()
        out.obj = self.obj.copy()
        out.pen = self.pen
        return out

    def key(self):
        return (tuple(int(s) for s in self.sizes),
                tuple(int(v) for r in range(self.d1) for v in self.row(r)))


@dataclass
class Spec:
    """The slice of core.ProblemConfig (core.py:112-151) the path reads."""

    kind: str
    d1: int
    d2: int
    n: int
    row_mode: str
    directions: tuple = (MIN,)
    weights: tuple = (1.0,)
    lb: int = 0
    ub: int = 0
    penalty_weight: float | None = None
    # Lexicographic comparison (core.py:92-106): (priority_order, tolerances);
    # None = Weighted with `weights` (core.py:80-90, engine.py:215-222)
    lex: tuple | None = None

    @property
    def m(self):
        return len(self.directions)


class Problem:
    spec: Spec

    def objective(self, i: int, sol: Sol) -> float:
        raise NotImplementedError

    def penalty(self, sol: Sol) -> float:
        return 0.0

    def matrices(self):
        """init_matrices (problems.py:62-64)."""
        return []

    def payload_nbytes(self) -> int:
        return sum(m.nbytes for m in self.matrices())


def evaluate(problem: Problem, sol: Sol):
    """problems.py:77-94 with validate=False (the engine's call)."""
    for i in range(problem.spec.m):
        sol.obj[i] = problem.objective(i, sol)
    sol.pen = float(problem.penalty(sol))
    return sol.obj, sol.pen


class Tsp(Problem):
    """builtins.py:53-77."""

    def __init__(self, dist):
        self.dist = np.asarray(dist, dtype=np.float64)
        n = self.dist.shape[0]
        self.n = n
        self.spec = Spec(PERM, 1, n, n, SINGLE)

    def objective(self, i, sol):
        t = sol.row(0)
        if len(t) < 2:
            return 0.0
        return float(self.dist[t[:-1], t[1:]].sum() + self.dist[t[-1], t[0]])

    def matrices(self):
        return [self.dist]


class Routing(Problem):
    """builtins.py:80-152 (CVRP); customers are values 0..n-1 at matrix c+1."""

    def __init__(self, dist, demands, capacity, vehicles, objectives=("distance",),
                 weights=None, lex=None):
        """objectives: names from ("distance", "vehicles") (builtins.py:80-116);
        weights: Weighted comparison weights (default: 1.0 per objective);
        lex: (priority_order, tolerances) for a Lexicographic comparison."""
        self.dist = np.asarray(dist, dtype=np.float64)
        self.demands = np.asarray(demands, dtype=np.float64)
        self.capacity = float(capacity)
        self.vehicles = int(vehicles)
        self.n = len(self.demands)
        self.names = tuple(objectives)
        m = len(self.names)
        w = tuple(float(x) for x in weights) if weights is not None and lex is None \
            else (1.0,) * m
        self.spec = Spec(PERM, self.vehicles, self.n, self.n, PARTITION, directions=(MIN,) * m,
                         weights=w, lex=lex)

    def route_len(self, route) -> float:
        if len(route) == 0:
            return 0.0
        nodes = route + 1
        total = self.dist[0, nodes[0]] + self.dist[nodes[-1], 0]
        if len(nodes) > 1:
            total += self.dist[nodes[:-1], nodes[1:]].sum()
        return float(total)

    def objective(self, i, sol):
        if self.names[i] == "vehicles":  # builtins.py:133
            return float(np.count_nonzero(sol.sizes))
        return sum(self.route_len(sol.row(r)) for r in range(sol.d1))

    def load_excess(self, sol) -> float:
        total = 0.0
        for r in range(sol.d1):
            load = self.demands[sol.row(r)].sum()
            total += max(0.0, float(load) - self.capacity)
        return total

    def penalty(self, sol):
        return self.load_excess(sol)

    def matrices(self):
        return [self.dist[1:, 1:]]

    def payload_nbytes(self):
        return self.dist.nbytes + self.demands.nbytes


class Vrptw(Routing):
    """builtins.py:155-190: capacity excess + sequential lateness."""

    def __init__(self, dist, demands, capacity, vehicles, ready, due, service, **mo):
        super().__init__(dist, demands, capacity, vehicles, **mo)
        self.ready = np.asarray(ready, dtype=np.float64)
        self.due = np.asarray(due, dtype=np.float64)
        self.service = np.asarray(service, dtype=np.float64)

    def lateness(self, sol) -> float:
        total = 0.0
        for r in range(sol.d1):
            route = sol.row(r)
            if len(route) == 0:
                continue
            t = self.ready[0]
            prev = 0
            for c in route:
                node = c + 1
                arrival = max(self.ready[node], t + self.dist[prev, node])
                total += max(0.0, arrival - self.due[node])
                t = arrival + self.service[node]
                prev = node
            total += max(0.0, t + self.dist[prev, 0] - self.due[0])
        return float(total)

    def penalty(self, sol):
        return self.load_excess(sol) + self.lateness(sol)

    def payload_nbytes(self):
        return super().payload_nbytes() + self.ready.nbytes + self.due.nbytes \
            + self.service.nbytes


class PriorityVrp(Routing):
    """builtins.py:193-210."""

    def __init__(self, dist, demands, capacity, vehicles, priorities, **mo):
        super().__init__(dist, demands, capacity, vehicles, **mo)
        self.prio = np.asarray(priorities, dtype=np.float64)

    def penalty(self, sol):
        v = 0
        for r in range(sol.d1):
            pr = self.prio[sol.row(r)]
            for p in range(len(pr)):
                v += int(np.count_nonzero(pr[p + 1:] > pr[p]))
        return self.load_excess(sol) + v


class NonlinearVrp(Routing):
    """builtins.py:213-237."""

    def objective(self, i, sol):
        if self.names[i] == "vehicles":
            return float(np.count_nonzero(sol.sizes))
        total = 0.0
        for r in range(sol.d1):
            route = sol.row(r)
            if len(route) == 0:
                continue
            load = 0.0
            prev = 0
            for c in route:
                node = c + 1
                total += self.dist[prev, node] * (1.0 + 0.3 * (load / self.capacity) ** 2)
                load += self.demands[c]
                prev = node
            total += self.dist[prev, 0] * (1.0 + 0.3 * (load / self.capacity) ** 2)
        return float(total)


class Knapsack(Problem):
    """builtins.py:240-262 (maximise value, penalty = weight excess)."""

    def __init__(self, weights, values, capacity):
        self.w = np.asarray(weights, dtype=np.float64)
        self.v = np.asarray(values, dtype=np.float64)
        self.capacity = float(capacity)
        self.n = len(self.w)
        self.spec = Spec(BINARY, 1, self.n, self.n, SINGLE, directions=(MAX,))

    def objective(self, i, sol):
        return float(self.v @ sol.row(0))

    def penalty(self, sol):
        return max(0.0, float(self.w @ sol.row(0)) - self.capacity)


class Qap(Problem):
    """builtins.py:265-290."""

    def __init__(self, flow, dist):
        self.flow = np.asarray(flow, dtype=np.float64)
        self.dist = np.asarray(dist, dtype=np.float64)
        self.n = self.flow.shape[0]
        self.spec = Spec(PERM, 1, self.n, self.n, SINGLE)

    def objective(self, i, sol):
        p = sol.row(0)
        return float((self.flow * self.dist[np.ix_(p, p)]).sum())

    def matrices(self):
        return [self.flow, self.dist]


class JspInt(Problem):
    """builtins.py:408-456: priority-decoded serial schedule generator."""

    def __init__(self, jobs):
        self.jobs = [[(int(m), int(d)) for m, d in ops] for ops in jobs]
        self.n_jobs = len(self.jobs)
        self.per_job = len(self.jobs[0])
        self.n_machines = 1 + max(m for ops in self.jobs for m, _ in ops)
        self.n_ops = self.n_jobs * self.per_job
        self.spec = Spec(INTEGER, 1, self.n_ops, self.n_ops, SINGLE, lb=0,
                         ub=self.n_ops - 1)

    def objective(self, i, sol):
        prio = sol.row(0)
        nxt = [0] * self.n_jobs
        job_free = [0.0] * self.n_jobs
        mach_free = [0.0] * self.n_machines
        span = 0.0
        for _ in range(self.n_ops):
            pick, pick_key = -1, None
            for j in range(self.n_jobs):
                k = nxt[j]
                if k >= self.per_job:
                    continue
                op = j * self.per_job + k
                key = (int(prio[op]), op)
                if pick_key is None or key < pick_key:
                    pick, pick_key = j, key
            m, d = self.jobs[pick][nxt[pick]]
            done = max(job_free[pick], mach_free[m]) + d
            job_free[pick] = done
            mach_free[m] = done
            nxt[pick] += 1
            span = max(span, done)
        return float(span)


def scalar_fitness(problem: Problem, sol: Sol, penalty_weight: float) -> float:
    """engine.py:215-222 via core.scalarize (core.py:292-307)."""
    spec = problem.spec
    total = 0.0
    for value, d, w in zip(sol.obj, spec.directions, spec.weights):
        total += w * (-value if d == MAX else value)
    return total + penalty_weight * sol.pen


def acceptance_delta(problem, cand: Sol, cur: Sol, penalty_weight: float) -> float:
    """engine.py:225-246: Weighted scalarised difference, or the Lexicographic
    difference on the first non-tied objective; penalties folded in both."""
    spec = problem.spec
    if spec.lex is None:
        return scalar_fitness(problem, cand, penalty_weight) - \
            scalar_fitness(problem, cur, penalty_weight)
    order, tol = spec.lex
    d = 0.0
    for i in order:
        diff = float(cand.obj[i]) - float(cur.obj[i])
        if abs(diff) <= tol[i]:
            continue
        if spec.directions[i] == MAX:
            diff = -diff
        d = diff
        break
    return d + penalty_weight * (cand.pen - cur.pen)


def compare(problem, a: Sol, b: Sol) -> int:
    """core.py:315-347: -1 a better, 0 equal, 1 b better (penalty first)."""
    fa_ok, fb_ok = a.pen == 0.0, b.pen == 0.0
    if fa_ok != fb_ok:
        return -1 if fa_ok else 1
    if not fa_ok and a.pen != b.pen:
        return -1 if a.pen < b.pen else 1
    spec = problem.spec
    if spec.lex is not None:  # core.py:338-346
        order, tol = spec.lex
        for i in order:
            if abs(a.obj[i] - b.obj[i]) <= tol[i]:
                continue
            low = spec.directions[i] == MIN
            if a.obj[i] < b.obj[i]:
                return -1 if low else 1
            return 1 if low else -1
        return 0
    fa, fb = _scal(problem, a), _scal(problem, b)
    if fa == fb:
        return 0
    return -1 if fa < fb else 1


def _scal(problem, sol):
    total = 0.0
    for value, d, w in zip(sol.obj, problem.spec.directions, problem.spec.weights):
        total += w * (-value if d == MAX else value)
    return total


def validate(problem: Problem, sol: Sol) -> bool:
    """Structural validity (core.py:212-274), boolean form."""
    s = problem.spec
    if sol.data.shape != (s.d1, s.d2) or np.any(sol.sizes < 0) or np.any(sol.sizes > s.d2):
        return False
    if s.kind == PERM:
        if s.row_mode == SINGLE:
            return sorted(sol.row(0).tolist()) == list(range(s.n))
        if s.row_mode == MULTI_FIXED:
            return all(sorted(sol.row(r).tolist()) == list(range(s.n)) for r in range(s.d1))
        return sorted(sol.flat().tolist()) == list(range(s.n))
    if s.kind == BINARY:
        return all(set(sol.row(r).tolist()) <= {0, 1} for r in range(s.d1))
    return all(((sol.row(r) >= s.lb) & (sol.row(r) <= s.ub)).all() for r in range(s.d1))


class Custom(Problem):
    """A user-defined single-row problem (the CUDA-snippet path of
    `solve_custom`; reference ProblemDefinition callbacks,
    problems.py:49-74).  `obj(row)` / `pen(row)` restate the test's CUDA snippet
    in Python with the same arithmetic order (test infrastructure only)."""

    def __init__(self, kind, n, obj, pen=None, lb=0, ub=0, maximize=False, mats=(),
                 weights=None, lex=None):
        # obj: one function or a list of two (core.py:69-106: per-objective
        # direction and weight; lex = (priority_order, tolerances))
        self.n = n
        objs = list(obj) if isinstance(obj, (list, tuple)) else [obj]
        maxes = [maximize] * len(objs) if isinstance(maximize, bool) else list(maximize)
        self.spec = Spec(kind, 1, n, n, SINGLE,
                         directions=tuple(MAX if mx else MIN for mx in maxes),
                         weights=tuple(weights) if weights else (1.0,) * len(objs),
                         lb=lb, ub=ub, lex=lex)
        self._objs, self._pen = objs, pen
        self._mats = [np.asarray(m, np.float64) for m in mats]

    def objective(self, i, sol):
        return float(self._objs[i](sol.row(0)))

    def penalty(self, sol):
        return float(self._pen(sol.row(0))) if self._pen is not None else 0.0

    def matrices(self):
        return list(self._mats)


class Assignment(Problem):
    """builtins.py:293-319."""

    def __init__(self, cost):
        self.cost = np.asarray(cost, dtype=np.float64)
        self.n = self.cost.shape[0]
        self.spec = Spec(PERM, 1, self.n, self.n, SINGLE)

    def objective(self, i, sol):
        return float(self.cost[np.arange(self.n), sol.row(0)].sum())

    def matrices(self):
        return [self.cost]


class GraphColoring(Problem):
    """builtins.py:322-350."""

    def __init__(self, num_vertices, edges, num_colors):
        self.n = int(num_vertices)
        self.eu = np.array([u for u, _ in edges], dtype=np.int64)
        self.ev = np.array([v for _, v in edges], dtype=np.int64)
        self.spec = Spec(INTEGER, 1, self.n, self.n, SINGLE, lb=0, ub=int(num_colors) - 1)

    def objective(self, i, sol):
        c = sol.row(0)
        return float(np.count_nonzero(c[self.eu] == c[self.ev]))


class BinPacking(Problem):
    """builtins.py:353-373."""

    def __init__(self, sizes, capacity):
        self.sizes = np.asarray(sizes, dtype=np.float64)
        self.capacity = float(capacity)
        self.n = len(self.sizes)
        self.spec = Spec(INTEGER, 1, self.n, self.n, SINGLE, lb=0, ub=self.n - 1)

    def objective(self, i, sol):
        return float(len(np.unique(sol.row(0))))

    def penalty(self, sol):
        loads = np.bincount(sol.row(0), weights=self.sizes, minlength=self.n)
        return float(np.maximum(loads - self.capacity, 0.0).sum())


class LoadBalancing(Problem):
    """builtins.py:376-394."""

    def __init__(self, durations, num_machines):
        self.d = np.asarray(durations, dtype=np.float64)
        self.m = int(num_machines)
        self.n = len(self.d)
        self.spec = Spec(INTEGER, 1, self.n, self.n, SINGLE, lb=0, ub=self.m - 1)

    def objective(self, i, sol):
        return float(np.bincount(sol.row(0), weights=self.d, minlength=self.m).max())


class JspPerm(Problem):
    """builtins.py:459-516: row m orders the jobs on machine m; the decoder
    sweeps the machines until no head operation can start, penalising
    operations left unscheduled by a cyclic wait."""

    def __init__(self, jobs):
        self.jobs = [[(int(m), int(d)) for m, d in ops] for ops in jobs]
        self.n_jobs, self.per_job = len(self.jobs), len(self.jobs[0])
        self.n_mach = 1 + max(m for ops in self.jobs for m, _ in ops)
        self.spec = Spec(PERM, self.n_mach, self.n_jobs, self.n_jobs, MULTI_FIXED)

    def decode(self, sol):
        ptr = [0] * self.n_mach
        nxt = [0] * self.n_jobs
        javail = [0.0] * self.n_jobs
        mavail = [0.0] * self.n_mach
        done_ops, total, span = 0, self.n_jobs * self.per_job, 0.0
        moved = True
        while moved and done_ops < total:
            moved = False
            for m in range(self.n_mach):
                if ptr[m] >= self.n_jobs:
                    continue
                j = int(sol.data[m, ptr[m]])
                k = nxt[j]
                if k >= self.per_job or self.jobs[j][k][0] != m:
                    continue
                end = max(javail[j], mavail[m]) + self.jobs[j][k][1]
                javail[j] = mavail[m] = end
                nxt[j] += 1
                ptr[m] += 1
                done_ops += 1
                span = max(span, end)
                moved = True
        return span, total - done_ops

    def objective(self, i, sol):
        return float(self.decode(sol)[0])

    def penalty(self, sol):
        return float(self.decode(sol)[1])


class BinarySchedule(Problem):
    """builtins.py:519-545: worker x shift 0/1 matrix; cost sum (numpy over the
    whole matrix), penalty = uncovered requirement per shift."""

    def __init__(self, cost, requirements):
        self.cost = np.asarray(cost, dtype=np.float64)
        self.req = np.asarray(requirements, dtype=np.float64)
        w, sh = self.cost.shape
        self.spec = Spec(BINARY, w, sh, w * sh, MULTI_FIXED)

    def objective(self, i, sol):
        return float((self.cost * sol.data).sum())

    def penalty(self, sol):
        return float(np.maximum(self.req - sol.data.sum(axis=0), 0.0).sum())
