"""Device island exchange (go_engine_export_elites / import_elites) against the
oracle's migrate() (engine.py:483-521): two engines on one GPU play two ranks;
their gathered records are imported by each and the resulting populations
must equal the reference rule applied to the two islands."""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2603_19163_b200 as G
from oracle import engine as OE
from oracle import problems as OP
from oracle.rng import STREAMS
from paper_2603_19163_b200 import _native as N
from paper_2603_19163_b200 import instances as I
from paper_2603_19163_b200.engine import DeviceRun, derived_rng

pytestmark = pytest.mark.gpu


def _pop_as_oracle(dr, ref):
    out = []
    for s in dr.population():
        o = OP.Sol(s.data, s.dim2_sizes, 1)
        OP.evaluate(ref, o)
        assert o.obj[0] == s.objectives[0]
        out.append(o)
    return out


@pytest.mark.parametrize("strategy,event,top_n", [("ring", 0, 1), ("global_top_n", 1, 2),
                                                  ("hybrid", 3, 3)])
def test_import_matches_reference_migration(strategy, event, top_n):
    d = I.tsp_random(30, 3)
    prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=d))
    ref = OP.Tsp(d)
    seed = 77
    drs = []
    for rank in range(2):
        cfg = G.EngineConfig(population=5, team_size=32, seed=seed, evolver_offset=rank << 20)
        dr = DeviceRun(prob, cfg, seed, init_rng=derived_rng(seed, 2, rank))
        dr.run(20, None)
        drs.append(dr)
    pops = [_pop_as_oracle(dr, ref) for dr in drs]
    before = [dr.best().objectives[0] for dr in drs]
    cur_best = min(s.obj[0] for p in pops for s in p)
    rb = C.c_int64()
    N.check(drs[0].lib.go_elite_record_bytes(drs[0].engine, C.byref(rb)))
    bufs = [torch.zeros(top_n * rb.value, dtype=torch.uint8, device="cuda") for _ in drs]
    for dr, b in zip(drs, bufs):
        N.check(dr.lib.go_engine_export_elites(dr.engine, C.c_void_p(b.data_ptr()), top_n))
        N.check(dr.lib.go_engine_sync(dr.engine))
    gathered = torch.cat(bufs)
    for rank, dr in enumerate(drs):
        N.check(dr.lib.go_engine_import_elites(dr.engine, C.c_void_p(gathered.data_ptr()), 2,
                                               rank, top_n, N.MIG[strategy], event))
    strat = strategy
    if strat == "hybrid":
        strat = "ring" if event % 2 == 0 else "global_top_n"
    OE.migrate(ref, pops, strat, STREAMS["philox"](seed, 3, event), top_n)
    for dr, pop in zip(drs, pops):
        got = [s.row(0).tolist() for s in dr.population()]
        assert got == [s.row(0).tolist() for s in pop]
    for dr, b0 in zip(drs, before):  # gathered bests refresh the global best (elite source)
        assert dr.best().objectives[0] == min(b0, cur_best)
        dr.close()


def _rank_main(rank, world, port, q, device_init=False):
    import os
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)  # ranks share cuda:0
    d = I.tsp_random(40, 5)
    prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=d))
    res = G.run(prob, G.EngineConfig(population=8, team_size=32, max_generations=250, seed=3,
                                     distributed=True, device=0, device_init=device_init,
                                     islands=G.IslandsConfig(count=world, migration="hybrid",
                                                             interval=50, top_n=2)))
    o = OP.Tsp(d)
    phi = o.objective(0, OP.Sol(res.best.data, res.best.dim2_sizes))
    q.put((rank, res.generations_completed, res.device["migration_events"], res.objectives[0],
           phi, res.device["winner_rank"]))
    dist.destroy_process_group()


@pytest.mark.parametrize("device_init", [False, True])
def test_run_distributed_two_ranks_one_gpu(device_init):
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q, device_init)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, g0, e0, b0, phi0, w0), (_, g1, e1, b1, phi1, w1) = out
    assert g0 == g1 == 250 and e0 == e1 == 5
    assert b0 == b1 == phi0 == phi1 and w0 == w1
