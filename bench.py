"""Benchmark: move evaluations / s and % gap @30 s on the pcb442-shaped TSP
(BASELINE.json metric; config C2: 26x17 lattice, known optimum 44,200, with
the user-registered tsp-delta operators compiled by NVRTC).

    python bench.py [--gpus N] [--steps K] [--warmup W]          # our engine
    python bench.py --impl reference [...]                         # CPU reference arm

A step = one evolve chunk of --gens-per-step generations (one AOS interval)
for the whole population, inputs resident in HBM; L2 is flushed (a 256 MiB
write on the engine's stream) between timed steps.  `value` is device-timed
(CUDA events on the engine stream, max over ranks); `e2e` is the same metric
through the C ABI with host buffers (population H2D + run + population D2H
per step).  Multi-GPU: one process per GPU, independent islands with
disjoint Philox streams (weak scaling, no data-path collective).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "move evals/sec and % gap @30s on TSP-442 shape at 1/2/4/8 B200 vs CPU ref"


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), "measured", d
    return 6650.0, "fallback", {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}",
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def ncu_traffic():
    """DRAM bytes per evolve launch from the committed ncu --set full capture
    (profiles/r01_ncu_traffic.json), or None."""
    p = ROOT / "profiles" / "r01_ncu_traffic.json"
    try:
        return json.loads(p.read_text())["dram_bytes_per_launch"]
    except (OSError, ValueError, KeyError):
        return None


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def other_configs(G, I, local, steps=5, gps=10):
    """Device throughput on the other BASELINE shapes (C1, C3, C4, C5a, C5b):
    a few 10-generation steps each with the B200 population rule."""
    vd = I.vrptw_solomon_like()
    f, dq = I.qap_random(100, 100)
    w, v, cap = I.knapsack_random(1000, 1000)
    probs = {
        "C1 TSP n=51 (nint)": G.builtin_problem("tsp", G.InstanceData(
            distance_matrix=I.tsp_random(51, 51))),
        "C3 VRPTW n=100, 25 vehicles": G.builtin_problem("vrptw", G.InstanceData(
            distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity,
            vehicles=vd.vehicles, ready_times=vd.ready, due_times=vd.due,
            service_times=vd.service)),
        "C4 QAP n=100": G.builtin_problem("qap", G.InstanceData(flow_matrix=f,
                                                                distance_matrix=dq)),
        "C5a JSP-int 20x15": G.builtin_problem("jsp_int", G.InstanceData(
            jobs=I.jsp_random(20, 15, 2015))),
        "C5b knapsack n=1000": G.builtin_problem("knapsack", G.InstanceData(
            weights=w, values=v, capacity=cap)),
    }
    out = {}
    for name, prob in probs.items():
        dr = G.DeviceRun(prob, G.EngineConfig(device=local), 42)
        done = 0
        for _ in range(2):
            done += gps
            dr.run(done, None)
        ms = 0.0
        for _ in range(steps):
            done += gps
            ms += dr.run(done, None).device_ms
        evals = dr.pop_size * 128 * gps * steps
        out[name] = {"move_evals_per_s": evals / (ms / 1e3), "population": dr.pop_size,
                     "ms_per_step": ms / steps, "smem_bytes": dr.smem_bytes,
                     "layout": dr.layout, "best_after": float(dr.best().objectives[0])}
        dr.close()
    return out


# ---------------------------------------------------------------------------
def run_ours(args):
    import ctypes as C

    import numpy as np
    import torch

    import paper_2603_19163_b200 as G
    from paper_2603_19163_b200 import _native as N
    from paper_2603_19163_b200 import instances as I

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl")
    d, opt = I.tsp_lattice()
    prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=d))
    ops = G.tsp_delta_operators()
    cfg = G.EngineConfig(team_size=args.team_size, seed=args.seed, custom_operators=ops,
                         device=local, population=args.population or None,
                         islands=G.IslandsConfig(count=world, migration="hybrid", interval=100))
    island = None
    if world > 1:  # ranks are islands: elite records all-gathered over NCCL every 100 gens
        from paper_2603_19163_b200 import islands as ISL
        island = ISL.DeviceIsland(prob, cfg, cfg.seed, rank)
        dr = island.dr
        rec = island.record_bytes
        send = island.buffer(rec)
        recv = island.buffer(world * rec)
        events = 0
    else:
        dr = G.DeviceRun(prob, cfg, cfg.seed)
    P, T = dr.pop_size, cfg.team_size
    gps = args.gens_per_step
    stream = C.c_void_p()
    N.check(dr.lib.go_engine_stream(dr.engine, C.byref(stream)))
    tstream = torch.cuda.ExternalStream(stream.value, device=torch.device("cuda", local))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    done = 0
    for _ in range(args.warmup):
        done += gps
        dr.run(done, None)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    dev_ms = evolve_ms = 0.0
    launches = evolve_launches = reads_pos = reads_elem = 0
    st = None
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(tstream):
                flush.random_(0, 255)  # L2 flush outside the timed events
                ev0.record(tstream)
            done += gps
            st = dr.run(done, None)
            if island is not None and done % 100 == 0:  # exchange inside the timed region
                ISL.exchange_round(island, world, rank, 1, 2, events, torch.distributed, send,
                                   recv)
                events += 1
                launches += 2
            with torch.cuda.stream(tstream):
                ev1.record(tstream)
            ev1.synchronize()
            dev_ms += ev0.elapsed_time(ev1)
            evolve_ms += st.evolve_ms
            launches += st.kernel_launches
            evolve_launches += st.evolve_launches
            reads_pos += st.reads_pos
            reads_elem += st.reads_elem
    torch.cuda.synchronize()
    gens_timed = args.steps * gps
    evals_local = P * T * gens_timed
    t_max = dev_ms
    evals_all = evals_local
    if world > 1:
        tt = torch.tensor([dev_ms], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_max = float(tt.item())
        ev = torch.tensor([evals_local], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(ev)
        evals_all = float(ev.item())
    value = evals_all / (t_max / 1e3)

    # ---- e2e through the C ABI with host buffers -----------------------------
    genes = np.zeros((P, dr.cfg.d2), dtype=np.int32)
    sizes = np.zeros((P, 1), dtype=np.int32)
    obj = np.zeros(P)
    pen = np.zeros(P)
    N.check(dr.lib.go_engine_get_population(dr.engine, N.iptr(genes), N.iptr(sizes),
                                            N.dptr(obj), N.dptr(pen)))
    if world > 1:
        torch.distributed.barrier()
    e2e_steps = max(3, args.steps // 2)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        N.check(dr.lib.go_engine_set_population(dr.engine, N.iptr(genes), N.iptr(sizes),
                                                N.dptr(obj), N.dptr(pen)))
        dr.run(gps, None)
        N.check(dr.lib.go_engine_get_population(dr.engine, N.iptr(genes), N.iptr(sizes),
                                                N.dptr(obj), N.dptr(pen)))
    e2e_wall = time.perf_counter() - t0
    if world > 1:
        tt = torch.tensor([e2e_wall], dtype=torch.float64, device=f"cuda:{local}")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_wall = float(tt.item())
    e2e_value = world * P * T * gps * e2e_steps / e2e_wall
    h2d = genes.nbytes + sizes.nbytes + obj.nbytes + pen.nbytes
    dr.close()
    if island is not None:
        torch.distributed.barrier()

    # ---- % gap at the 30 s budget through the public run() ------------------------
    gap = None
    gap_info = {}
    if args.gap_seconds > 0:
        res = G.run(prob, G.EngineConfig(team_size=args.team_size, seed=args.seed + 7,
                                         custom_operators=ops, device=local,
                                         time_limit_seconds=args.gap_seconds,
                                         max_generations=10 ** 9, distributed=world > 1,
                                         device_init=True,
                                         islands=G.IslandsConfig(count=world, migration="hybrid",
                                                                 interval=100)),
                    best_known=opt)
        gaps = [res.gap_pct]
        gap = min(gaps)
        gap_info = {"gap_pct_30s": gap, "gap_pct_30s_per_rank": gaps,
                    "best_30s": res.objectives[0], "generations_30s": res.generations_completed,
                    "move_evals_per_s_30s": (res.device.get("lane_evals", 0) / res.elapsed_seconds)
                    if world == 1 else None,
                    "elapsed_30s": res.elapsed_seconds,
                    "final_weights_30s": {e["name"]: round(e["weight"], 4)
                                          for e in res.final_weights["sequences"]},
                    "k_weights_30s": [round(x, 4) for x in res.final_weights["k_steps"]]}
        # time to the known optimum (44,200) through the same API: target_objective stops
        # the run at the chunk where the global best reaches it (engine.py:712-713)
        rt = G.run(prob, G.EngineConfig(team_size=args.team_size, seed=args.seed + 7,
                                        custom_operators=ops, device=local,
                                        time_limit_seconds=args.gap_seconds,
                                        target_objective=opt, max_generations=10 ** 9,
                                        distributed=world > 1, device_init=True,
                                        islands=G.IslandsConfig(count=world, migration="hybrid",
                                                                interval=100)),
                   best_known=opt)
        hit = rt.gap_pct == 0.0
        gap_info.update({"time_to_optimum_s": rt.elapsed_seconds if hit else None,
                         "generations_to_optimum": rt.generations_completed if hit else None})

    extra = other_configs(G, I, local) if (args.other_configs and world == 1) else None
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    hbm, src, pk = peaks()
    alg_bytes = reads_pos * 2 + reads_elem * (st.elem_bytes if st else 2)
    achieved_gbs = alg_bytes / (evolve_ms / 1e3) / 1e9 if evolve_ms > 0 else 0.0
    clocks = clk.summary()
    info = N.device_info(local)
    sm_mhz = clocks.get("sm_mhz") or pk.get("clocks_under_load", {}).get("sm_mhz_median", 1965.0)
    smem_peak = info.sm_count * 128 * sm_mhz * 1e6 / 1e9
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import cpu_bench
        procs = cpu_cores() if args.cpu_procs == 0 else args.cpu_procs
        cb = cpu_bench.throughput(d, procs, pop=8, team=128, gens=args.cpu_gens)
        cpu = {"value": cb["value"], "unit": "move evals/s", "cores": procs, "kind": "port",
               "sample": f"oracle engine (== reference run(), MT19937) on C2 with tsp-delta, full "
                         f"reference registry: {procs} processes x P=8 x T=128 x "
                         f"{args.cpu_gens} generations ({cb['evals']} evals in "
                         f"{cb['wall_s']:.1f} s)"}
    out = {
        "metric": METRIC, "value": value, "unit": "move evals/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int16 genes / int16 distances, int64 deltas",
        "data": "synthetic (seeded 26x17 lattice, permuted labels, TSPLIB nint)",
        "config": {"workload": "C2 pcb442-shaped lattice TSP n=442 + user tsp-delta ops (NVRTC)",
                   "population_per_gpu": P, "team_size": T, "generations_per_step": gps,
                   "layout": "int16 packed triangle in shared memory",
                   "l2": "flushed between timed steps (256 MiB write)",
                   "parallelism": f"islands x{world}" + (" (NCCL elite all_gather every 100 "
                                                         "generations, hybrid migration)"
                                                         if world > 1 else "")},
        "e2e": {"value": e2e_value, "unit": "move evals/s", "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(h2d),
                "path": "go_engine_set_population(host) + go_engine_run + "
                        "go_engine_get_population(host) per step",
                "l2": "not flushed between e2e steps (host copies take the flush's place); the "
                      "device-timed value flushes L2, so its steps start with cold L2 and "
                      "instruction fetch"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": hbm, "unit": "GB/s",
                     "frac": achieved_gbs / hbm, "traffic": ncu_traffic(),
                     "peak_source": src, "kernel": "go_evolve_tsp_jit",
                     "evolve_ms": evolve_ms, "evolve_launches": int(evolve_launches),
                     "algorithmic_bytes": int(alg_bytes),
                     "note": "instance and solutions are shared-memory resident; see smem"},
        "roofline_smem": {"achieved": achieved_gbs, "peak": smem_peak, "unit": "GB/s",
                          "frac": achieved_gbs / smem_peak,
                          "peak_formula": f"{info.sm_count} SM x 128 B/clk x {sm_mhz} MHz"},
        "clocks": clocks,
        "communicator": ({"backend": torch.distributed.get_backend(), "world": world,
                          "nccl_version": ".".join(map(str, torch.cuda.nccl.version())),
                          "exchange": "elite all_gather every 100 generations"}
                         if world > 1 else None),
        "cpu_baseline": cpu,
        **gap_info,
        "other_configs": extra,
    }
    print(json.dumps(out))
    if world > 1:
        torch.distributed.destroy_process_group()


# ---------------------------------------------------------------------------
def run_reference(args):
    """The reference's own algorithm on the host cores: the oracle in MT mode
    reproduces genopt.run() bit-for-bit (pinned by tests/golden)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from oracle import cpu_bench
    from paper_2603_19163_b200 import instances as I
    d, opt = I.tsp_lattice()
    procs = cpu_cores() if args.cpu_procs == 0 else args.cpu_procs
    vals = []
    t_all = time.perf_counter()
    for _ in range(args.warmup):
        cpu_bench.throughput(d, procs, pop=4, team=128, gens=1)
    for _ in range(args.steps):
        vals.append(cpu_bench.throughput(d, procs, pop=8, team=128, gens=args.cpu_gens))
    value = sum(v["evals"] for v in vals) / sum(v["wall_s"] for v in vals)
    gap = {}
    if args.gap_seconds > 0:
        g = cpu_bench.gap_at(d, args.gap_seconds, procs, opt)
        gap = {"gap_pct_30s": g["best_gap_pct"], "median_gap_pct_30s": g["median_gap_pct"],
               "move_evals_per_s_30s": g["evals_per_s"]}
    out = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "move evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(v["wall_s"] for v in vals) / max(1, len(vals)),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded 26x17 lattice, permuted labels, TSPLIB nint)",
        "config": {"workload": "C2 pcb442-shaped lattice TSP n=442 + user tsp-delta ops",
                   "population_per_process": 8, "team_size": 128,
                   "generations_per_step": args.cpu_gens},
        "cpu_baseline": {"value": value, "unit": "move evals/s", "cores": procs, "kind": "port",
                         "sample": f"{procs} processes x P=8 x T=128 x {args.cpu_gens} "
                                   "generations per step, oracle MT mode == reference run()"},
        "e2e": {"value": value, "unit": "move evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": time.perf_counter() - t_all,
        **gap,
    }
    print(json.dumps(out))


def free_port() -> int:
    import socket
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch(n: int, argv: list[str]) -> int:
    """`bench.py --gpus N` outside torchrun: re-execute this script as N ranks
    (one process per GPU) under torch.distributed.run on 127.0.0.1, the same
    launch the driver uses, and return the launcher's exit status."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={free_port()}",
           str(Path(__file__).resolve()), *argv]
    return subprocess.call(cmd)


def selftest_dist(args):
    """Launcher / timing-protocol check without GPUs (gloo): every rank does a
    fixed amount of host work between barriers, the time is the MAX over ranks
    and rank 0 prints one line with the whole-job value (tests/test_bench_cpu.py)."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
        dist.barrier()
    t0 = time.perf_counter()
    units = 0
    for _ in range(args.steps):
        x = 0
        for i in range(20000):
            x += i * i
        units += 20000
    dt = time.perf_counter() - t0
    t = torch.tensor([dt], dtype=torch.float64)
    u = torch.tensor([float(units)], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(u)
        dist.barrier()
    if rank == 0:
        print(json.dumps({"metric": "selftest units/s", "value": float(u.item() / t.item()),
                          "n_gpus": world, "steps": args.steps, "ranks_seen": world,
                          "backend": "gloo" if world > 1 else None}))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--gens-per-step", type=int, default=10)
    ap.add_argument("--team-size", type=int, default=128)
    ap.add_argument("--population", type=int, default=0)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--gap-seconds", type=float, default=30.0)
    ap.add_argument("--cpu-gens", type=int, default=4)
    ap.add_argument("--cpu-procs", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--other-configs", type=int, default=1,
                    help="also measure C1/C3/C4/C5 device throughput (N=1 only)")
    ap.add_argument("--selftest-dist", action="store_true",
                    help="check the N-rank launcher and max-over-ranks timing on CPU (gloo)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args.gpus, sys.argv[1:]))
    _, world, _ = dist_env()
    if world != args.gpus and "WORLD_SIZE" in os.environ:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using WORLD_SIZE",
              file=sys.stderr)
    if args.selftest_dist:
        selftest_dist(args)
        return
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
