"""Multi-GPU island protocol on CPU: world_size 2 over gloo (127.0.0.1) with
a numpy island standing in for the device engine.  Covers the exchange loop
(islands.run_island_loop), stop agreement, record round trips and the
comparison-best reduction (islands.best_over_ranks)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2603_19163_b200 as G
from paper_2603_19163_b200 import islands as ISL


class NumpyIsland:
    """P members of a permutation problem with (pen, scal) = (0, cost(genes))."""

    def __init__(self, rank, P=6, n=12):
        self.rng = np.random.default_rng(100 + rank)
        self.P, self.n = P, n
        self.genes = np.stack([self.rng.permutation(n) for _ in range(P)]).astype(np.int16)
        self.w = np.arange(1, n + 1, dtype=np.float64)
        self.record_bytes = 16 + ((2 * n + 15) // 16) * 16
        self.gens = 0
        self.received = []

    def cost(self, g):
        return float(self.w @ g.astype(np.float64))

    def buffer(self, nbytes):
        return torch.zeros(nbytes, dtype=torch.uint8)

    def run(self, until, remaining):
        while self.gens < until:  # toy evolution: improving random swaps
            i = self.rng.integers(self.P)
            a, b = self.rng.choice(self.n, 2, replace=False)
            g = self.genes[i].copy()
            g[a], g[b] = g[b], g[a]
            if self.cost(g) < self.cost(self.genes[i]):
                self.genes[i] = g
            self.gens += 1
        return self.gens, False, None

    def order(self):
        return sorted(range(self.P), key=lambda i: (self.cost(self.genes[i]), i))

    def export(self, buf, top_n):
        raw = np.zeros(top_n * self.record_bytes, dtype=np.uint8)
        for d, i in enumerate(self.order()[:top_n]):
            rec = raw[d * self.record_bytes:(d + 1) * self.record_bytes]
            rec[:16] = np.frombuffer(np.array([self.cost(self.genes[i]), 0.0]).tobytes(), np.uint8)
            rec[16:16 + 2 * self.n] = np.frombuffer(self.genes[i].tobytes(), np.uint8)
        buf.copy_(torch.from_numpy(raw))

    def records(self, buf, count):
        raw = buf.numpy()
        out = []
        for d in range(count):
            rec = raw[d * self.record_bytes:(d + 1) * self.record_bytes]
            scal, pen = np.frombuffer(rec[:16].tobytes(), np.float64)
            genes = np.frombuffer(rec[16:16 + 2 * self.n].tobytes(), np.int16).copy()
            out.append((pen, scal, genes))
        return out

    def import_(self, buf, world, rank, top_n, strategy, event):
        recs = self.records(buf, world * top_n)
        if strategy == 2:
            strategy = 0 if event % 2 == 0 else 1
        if strategy == 0:  # ring: previous rank's best replaces our worst
            donor = recs[((rank - 1) % world) * top_n]
            order = self.order()
            worst, best = order[-1], order[0]
            if worst != best:
                self.genes[worst] = donor[2]
                self.received.append(donor[1])
        else:
            donors = sorted(range(len(recs)), key=lambda j: (recs[j][1], j))[:top_n]
            b = self.order()[0]
            slots = [i for i in range(self.P) if i != b]
            for j, d in enumerate(donors):
                self.genes[slots[(event + j) % len(slots)]] = recs[d][2]
                self.received.append(recs[d][1])

    def collective_stream(self):
        import contextlib
        return contextlib.nullcontext()

    def best(self):
        i = self.order()[0]
        s = G.Solution(self.genes[i][None, :].astype(np.int64), [self.n], 1)
        s.objectives[0] = self.cost(self.genes[i])
        s.penalty = 0.0
        return s


def _worker(rank, world, port, strategy, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    island = NumpyIsland(rank)
    cfg = G.EngineConfig(max_generations=450, islands=G.IslandsConfig(
        count=world, migration=strategy, interval=100, top_n=2))
    import time
    gens, events = ISL.run_island_loop(island, cfg, dist, rank, world, time.perf_counter())
    bests = [None] * world
    dist.all_gather_object(bests, island.best().objectives[0])
    prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=np.zeros((12, 12))))
    best, win = ISL.best_over_ranks(prob, island.best(), dist, world)
    out.put((rank, gens, events, len(island.received), bests, float(best.objectives[0]), win,
             sorted(best.data[0].tolist())))
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("strategy", ["ring", "global_top_n", "hybrid"])
def test_two_rank_island_exchange_over_gloo(strategy):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, strategy, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, g0, e0, n0, b0, best0, w0, genes0), (r1, g1, e1, n1, b1, best1, w1, genes1) = res
    assert g0 == g1 == 450 and e0 == e1 == 4          # exchanges after gens 100..400
    assert n0 > 0 and n1 > 0                           # both islands received migrants
    assert best0 == best1 == min(b0)                   # comparison-best over ranks, agreed
    assert w0 == w1 and genes0 == genes1 == list(range(12))


def _mo_worker(rank, world, port, out):
    """Two-objective CVRP (distance, vehicles) under Lexicographic vehicles-first:
    rank 0 has the shorter distance, rank 1 fewer vehicles — rank 1 must win and
    the returned objective vector must be rank 1's whole vector."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    xy = rng.uniform(0, 100, (7, 2))
    d = np.sqrt(((xy[:, None] - xy[None]) ** 2).sum(-1))
    prob = G.builtin_problem("cvrp", G.InstanceData(
        distance_matrix=d, demands=np.ones(6), capacity=6.0, vehicles=3,
        meta={"objectives": ("distance", "vehicles"),
              "comparison": G.Lexicographic((1, 0), (0.0, 0.0))}))
    cfg = prob.config()
    s = G.Solution(np.zeros((cfg.d1, cfg.d2), dtype=np.int64), np.zeros(cfg.d1, np.int64), 2)
    s.data[0, :6] = np.arange(6) if rank == 1 else [0, 1, 2, 0, 0, 0]
    s.dim2_sizes[0] = 6 if rank == 1 else 3
    if rank == 0:
        s.data[1, :3] = [3, 4, 5]
        s.dim2_sizes[1] = 3
    s.objectives[:] = [100.0, 2.0] if rank == 0 else [150.0, 1.0]
    s.penalty = 0.0
    best, win = ISL.best_over_ranks(prob, s, dist, world)
    out.put((rank, win, [float(x) for x in best.objectives], best.dim2_sizes.tolist()))
    dist.destroy_process_group()


def test_best_over_ranks_compares_whole_objective_vector():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, win, objs, sizes in res:
        assert win == 1 and objs == [150.0, 1.0] and sizes[0] == 6
