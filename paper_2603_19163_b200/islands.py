"""Multi-GPU island model: one process per GPU, each rank one island.

The reference's island model (engine.py:483-521, :730-743) partitions one
population into islands inside one process.  Here every GPU evolves its own
population (disjoint Philox evolver indices: rank * 2^20 + local index) and
every `islands.interval` generations the ranks exchange elites:

    export (device kernel: stable top_n records into a device buffer)
      -> all_gather of the fixed-size records (NCCL over NVLink on GPUs,
         gloo in the CPU tests)
      -> import (device kernel: the reference's ring / global_top_n / hybrid
         rule applied to this rank's island; gathered bests refresh the
         global best used by elite injection)

Stop decisions are agreed at every exchange (all_reduce MAX of a stop flag),
so every rank performs the same number of collectives.  The final result is
the comparison-best over ranks (engine.py:609-614).  AOS statistics stay per
GPU (the paper's multi-GPU mode is independent populations).
"""

from __future__ import annotations

import ctypes as C
import time
from dataclasses import replace

import numpy as np

from .core import A_BETTER, Direction, compare

RANK_STRIDE = 1 << 20   # evolver index offset per rank (disjoint lane streams)
STRATEGY = {"ring": 0, "global_top_n": 1, "hybrid": 2}


class DeviceIsland:
    """A rank's island backed by libcugenopt (DeviceRun) on its own GPU."""

    def __init__(self, problem, config, seed, rank):
        import torch

        from . import _native as N
        from .engine import DeviceRun, _STREAM_INIT, derived_rng
        self.N = N
        local = replace(config, islands=replace(config.islands, count=1),
                        evolver_offset=rank * RANK_STRIDE)
        self.dr = DeviceRun(problem, local, seed, init_rng=derived_rng(seed, _STREAM_INIT, rank),
                            init_salt=rank)
        rb = C.c_int64()
        N.check(self.dr.lib.go_elite_record_bytes(self.dr.engine, C.byref(rb)))
        self.record_bytes = rb.value
        self.device = torch.device("cuda", config.device)
        st = C.c_void_p()
        N.check(self.dr.lib.go_engine_stream(self.dr.engine, C.byref(st)))
        self.stream = torch.cuda.ExternalStream(st.value, device=self.device)

    def buffer(self, nbytes):
        import torch
        return torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    def run(self, until, remaining):
        st = self.dr.run(until, remaining)
        return int(st.generations), int(st.stopped_by) != 0, st

    def export(self, buf, top_n):
        self.N.check(self.dr.lib.go_engine_export_elites(self.dr.engine, C.c_void_p(buf.data_ptr()),
                                                        top_n))

    def import_(self, buf, world, rank, top_n, strategy, event):
        self.N.check(self.dr.lib.go_engine_import_elites(
            self.dr.engine, C.c_void_p(buf.data_ptr()), world, rank, top_n, strategy, event))

    def collective_stream(self):
        import torch
        return torch.cuda.stream(self.stream)

    def best(self):
        b = self.dr.best()
        return b

    def close(self):
        self.dr.close()


def exchange_round(island, world, rank, top_n, strategy, event, dist, send, recv):
    """One migration event: export -> all_gather -> import.  Device buffers
    go straight to NCCL; a gloo group (CPU tests, several ranks sharing one
    GPU) stages the few-KB records through host memory."""
    import torch
    island.export(send, top_n)
    with island.collective_stream():
        staged = send.is_cuda and dist.get_backend() != "nccl"
        src = send.cpu() if staged else send
        parts = [torch.empty_like(src) for _ in range(world)]
        dist.all_gather(parts, src)
        recv.copy_(torch.cat(parts))
    island.import_(recv, world, rank, top_n, strategy, event)


def _coll_device(dist, device):
    return device if dist.get_backend() == "nccl" else "cpu"


def agree_stop(local_stop, dist, device):
    import torch
    device = _coll_device(dist, device)
    t = torch.tensor([1 if local_stop else 0], dtype=torch.int32, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return bool(t.item())


def run_island_loop(island, config, dist, rank, world, t_start, device="cpu"):
    """The exchange loop shared by the device islands and the CPU protocol
    tests.  Returns (generations, migration events)."""
    isl = config.islands
    top_n = min(isl.top_n, 64)
    strategy = STRATEGY[isl.migration]
    send = island.buffer(top_n * island.record_bytes)
    recv = island.buffer(world * top_n * island.record_bytes)
    gens, events = 0, 0
    while True:
        target = min(config.max_generations, (gens // isl.interval + 1) * isl.interval)
        remaining = None
        if config.time_limit_seconds is not None:
            remaining = config.time_limit_seconds - (time.perf_counter() - t_start)
        timed_out = remaining is not None and remaining <= 0
        if not timed_out:
            gens, stopped, _ = island.run(target, remaining)
            timed_out = stopped and gens < target
        # a deadline on any rank ends the run for all (same collective count)
        if agree_stop(timed_out, dist, device):
            break
        if gens % isl.interval == 0:  # migration at the end of generation g (engine.py:730)
            exchange_round(island, world, rank, top_n, strategy, events, dist, send, recv)
            events += 1
        if gens >= config.max_generations:
            break
    return gens, events


def best_over_ranks(problem, best, dist, world, device="cpu"):
    """Comparison-best over ranks (engine.py:609-614): all_gather of each
    rank's (penalty, objective vector), then a broadcast of the winner's
    genes.  The whole vector is compared, so two-objective runs (routing
    distance + vehicles, Weighted or Lexicographic) pick the right rank."""
    import torch
    cfg = problem.config()
    device = _coll_device(dist, device)
    row = torch.tensor([best.penalty, *[float(x) for x in best.objectives]],
                       dtype=torch.float64, device=device)
    rows = [torch.zeros_like(row) for _ in range(world)]
    dist.all_gather(rows, row)
    vals = [r.cpu().numpy() for r in rows]
    win = 0
    for r in range(1, world):
        a, b = _as_sol(best, vals[r]), _as_sol(best, vals[win])
        if compare(a, b, cfg) == A_BETTER:
            win = r
    genes = torch.tensor(best.data.reshape(-1), dtype=torch.int64, device=device)
    sizes = torch.tensor(best.dim2_sizes, dtype=torch.int64, device=device)
    dist.broadcast(genes, src=win)
    dist.broadcast(sizes, src=win)
    out = _as_sol(best, vals[win])
    out.data = genes.cpu().numpy().reshape(best.data.shape)
    out.dim2_sizes = sizes.cpu().numpy()
    return out, win


def _as_sol(template, v):
    s = template.copy()
    s.penalty = float(v[0])
    s.objectives[:] = [float(x) for x in v[1:]]
    return s


def gap_pct(cfg, objectives, best_known):
    """RunResult.gap_pct as _run_single computes it: single objective,
    minimised, best_known given and non-zero."""
    if best_known is None or not best_known or cfg.num_objectives != 1 or \
            cfg.obj_defs[0].direction is not Direction.MINIMIZE:
        return None
    return (float(objectives[0]) - best_known) / best_known * 100.0


def run_distributed(problem, config, best_known=None):
    """`run()` across the ranks of an initialised torch.distributed NCCL group
    (one GPU per rank, e.g. launched with torchrun).  The ranks ARE the
    replicas of the paper's multi-GPU mode, so
    `replicas > 1` together with `distributed=True` is rejected.  As in
    _run_single, NVRTC compile time is reported apart from the budget
    (PAPER.md:811-812)."""
    import torch.distributed as dist

    from .engine import RunResult
    if config.replicas != 1:
        raise ValueError("distributed runs use one island per rank; replicas must be 1 "
                         "(use EngineConfig(replicas=N) without distributed=True instead)")
    rank, world = dist.get_rank(), dist.get_world_size()
    t_start = time.perf_counter()
    island = DeviceIsland(problem, config, config.seed, rank)
    jit = island.dr.jit_seconds
    try:
        gens, events = run_island_loop(island, config, dist, rank, world, t_start + jit,
                                       device=island.device)
        best, winner = best_over_ranks(problem, island.best(), dist, world, island.device)
        w, kw = island.dr.weights()
    finally:
        island.close()
    elapsed = time.perf_counter() - t_start - jit
    cfg = problem.config()
    echo = config.as_dict()
    echo["population_effective"] = island.dr.pop_size
    return RunResult(
        best=best, objectives=[float(v) for v in best.objectives], penalty=float(best.penalty),
        feasible=best.penalty == 0.0, gap_pct=gap_pct(cfg, best.objectives, best_known),
        generations_completed=gens,
        elapsed_seconds=elapsed, gens_per_sec=gens / elapsed if elapsed > 0 else 0.0,
        final_weights={"sequences": [{"id": e.id, "name": e.name, "weight": float(x)}
                                     for e, x in zip(island.dr.registry.entries, w)],
                       "k_steps": [float(x) for x in kw]},
        profile=island.dr.profile.as_dict(), config=echo, seed=config.seed,
        device={"rank": rank, "world": world, "migration_events": events,
                "winner_rank": winner, "population_per_rank": island.dr.pop_size,
                "jit_seconds": jit})
