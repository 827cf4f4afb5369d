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
    """DRAM bytes per evolve launch of the current kernel from its committed ncu
    --set full capture (profiles/r02_ncu_traffic.json, written by
    tools/ncu_traffic.py from the .ncu-rep of the same head), or None."""
    p = ROOT / "profiles" / "r02_ncu_traffic.json"
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


def best_known():
    """profiles/best_known.json: the reference values the gap figures use
    (exact optima and bounds from tools/bounds.py, best-known tours from long
    device runs, tools/best_known_runs.py)."""
    p = ROOT / "profiles" / "best_known.json"
    try:
        return json.loads(p.read_text())
    except (OSError, ValueError):
        return {}


def gap_of(value, ref, sense):
    if ref is None or value is None or not ref:
        return None
    return (value - ref) / abs(ref) * 100.0 if sense == "min" else (ref - value) / abs(ref) * 100.0


OTHER = {  # name -> label (BASELINE.json configs)
    "C1": "C1 random Euclidean TSP n=51 (nint)",
    "C2j": "C2j pcb442-shaped lattice with +-30 jitter + tsp-delta",
    "C3": "C3 VRPTW R101 fixture (100 customers, 25 vehicles)",
    "C4": "C4 QAP n=100",
    "C5a": "C5a JSP-int 20x15",
    "C5b": "C5b knapsack n=1000",
}


def other_configs(G, I, local, args, hbm, smem_peak, steps=5, gps=10):
    """The other BASELINE shapes at N=1: device throughput with its roofline,
    gap at the wall-clock budget through the public run(), and the reference
    beside it on the host cores — its gap@budget runs in a background process
    pool during the device's own budget, its steady-state throughput on a
    bounded sample afterwards."""
    from baseline import refbench as R
    table = I.baseline_instances()
    bk = best_known()
    procs = cpu_cores() if args.cpu_procs == 0 else args.cpu_procs
    out = {}
    for name, label in OTHER.items():
        if args.only and name not in args.only.split(","):
            continue
        kind, inst, opt = table[name]
        prob = G.builtin_problem(kind, inst)
        ops = G.tsp_delta_operators() if name == "C2j" else ()
        ref = bk.get(name, {})
        sense = ref.get("sense", "min")
        known = ref.get("optimum", ref.get("best_known"))
        dr = G.DeviceRun(prob, G.EngineConfig(device=local, custom_operators=ops), args.seed)
        done = 0
        for _ in range(2):
            done += gps
            dr.run(done, None)
        ms = emsum = 0.0
        rp = re_ = 0
        st = None
        for _ in range(steps):
            done += gps
            st = dr.run(done, None)
            ms += st.device_ms
            emsum += st.evolve_ms
            rp += st.reads_pos
            re_ += st.reads_elem
        evals = dr.pop_size * dr.config.team_size * gps * steps
        alg = rp * 2 + re_ * st.elem_bytes
        ach = alg / (emsum / 1e3) / 1e9 if emsum > 0 else 0.0
        row = {"workload": label, "move_evals_per_s": evals / (ms / 1e3),
               "population": dr.pop_size, "team_size": dr.config.team_size,
               "ms_per_step": ms / steps, "generations_per_step": gps,
               "smem_bytes": dr.smem_bytes, "layout": dr.layout, "teams_per_sm": dr.teams_per_sm,
               "roofline": {"bound": "smem (on-chip instance)", "achieved": ach, "unit": "GB/s",
                            "peak_hbm": hbm, "frac_hbm": ach / hbm, "peak_smem": smem_peak,
                            "frac_smem": ach / smem_peak, "algorithmic_bytes": int(alg),
                            "evolve_ms": emsum}}
        dr.close()
        if args.other_gap_seconds > 0:
            import threading
            cpu_gap = {}
            th = None
            if not args.no_cpu_baseline:
                th = threading.Thread(target=lambda: cpu_gap.update(R.gap_at(
                    name, args.other_gap_seconds, procs, known, sense)), daemon=True)
                th.start()
            res = G.run(prob, G.EngineConfig(device=local, seed=args.seed + 7,
                                             custom_operators=ops, device_init=True,
                                             time_limit_seconds=args.other_gap_seconds,
                                             max_generations=10 ** 9))
            if th is not None:
                th.join()
            val = float(res.objectives[0]) if res.penalty == 0.0 else None
            if "penalty_lower_bound" in ref:  # no zero-penalty solution exists (C3's R101)
                row.update({"penalty": float(res.penalty), "objective": float(res.objectives[0]),
                            "penalty_lower_bound": ref["penalty_lower_bound"],
                            "penalty_excess_pct": gap_of(float(res.penalty),
                                                         ref["penalty_lower_bound"], "min")})
            row.update({"gap_seconds": args.other_gap_seconds, "best": val,
                        "gap_pct": gap_of(val, known, sense),
                        "gap_reference": {k: v for k, v in ref.items()},
                        "generations": res.generations_completed,
                        "move_evals_per_s_run": res.device["lane_evals"] / res.elapsed_seconds})
            if "lower_bound" in ref:
                row["gap_pct_vs_lower_bound"] = gap_of(val, ref["lower_bound"], "min")
            if cpu_gap:
                cpu_gap["gap_pct_vs_reference"] = gap_of(cpu_gap.get("best"), known, sense)
                row["cpu_gap"] = cpu_gap
        if not args.no_cpu_baseline:
            tb = R.steady_throughput(name, procs, pop=8, team=128, warm=2, gens=2)
            row["cpu_baseline"] = {"value": tb["value"], "unit": "move evals/s", "cores": procs,
                                   "kind": tb["kind"], "cpu_model": R.cpu_model(),
                                   "sample": f"{procs} processes x genopt.run(P=8, T=128), "
                                             f"generations 3-4 timed ({tb['evals']} evals)"}
        out[name] = row
        print(f"[bench] {name}: {json.dumps(row)}", file=sys.stderr, flush=True)
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

    hbm, src, pk = peaks()
    alg_bytes = reads_pos * 2 + reads_elem * (st.elem_bytes if st else 2)
    achieved_gbs = alg_bytes / (evolve_ms / 1e3) / 1e9 if evolve_ms > 0 else 0.0
    clocks = clk.summary()
    info = N.device_info(local)
    sm_mhz = clocks.get("sm_mhz") or pk.get("clocks_under_load", {}).get("sm_mhz_median", 1965.0)
    smem_peak = info.sm_count * 128 * sm_mhz * 1e6 / 1e9
    extra = other_configs(G, I, local, args, hbm, smem_peak) \
        if (args.other_configs and world == 1) else None
    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline:
        from baseline import refbench as R
        procs = cpu_cores() if args.cpu_procs == 0 else args.cpu_procs
        cb = R.steady_throughput("C2", procs, pop=8, team=128, warm=args.cpu_warm_gens,
                                 gens=args.cpu_gens)
        cpu = {"value": cb["value"], "unit": "move evals/s", "cores": procs, "kind": cb["kind"],
               "cpu_model": R.cpu_model(),
               "sample": f"{'genopt.run() (the unmodified reference)' if cb['kind'] == 'reference' else 'oracle port of genopt.run()'}"
                         f" on C2 with tsp-delta and its full registry: {procs} processes x "
                         f"P=8 x T=128, generations {args.cpu_warm_gens + 1}-"
                         f"{args.cpu_warm_gens + args.cpu_gens} timed ({cb['evals']} evals in "
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
    """The reference's own implementation on the host cores: genopt.run() of
    the unmodified reference package (baseline/_ref, tools/stage_reference.sh)
    in one process per core (its evolver threads are GIL-bound), same C2
    workload and registry; the oracle port stands in when it is absent.
    A step = one generation of every process, after `warmup` generations."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from baseline import refbench as R
    procs = cpu_cores() if args.cpu_procs == 0 else args.cpu_procs
    t_all = time.perf_counter()
    tb = R.steady_throughput("C2", procs, pop=8, team=128, warm=args.warmup, gens=args.steps)
    value = tb["value"]
    gap = {}
    if args.gap_seconds > 0:
        g = R.gap_at("C2", args.gap_seconds, procs, 44200.0, "min")
        gap = {"gap_pct_30s": g.get("gap_pct"), "median_gap_pct_30s": g.get("median_gap_pct"),
               "best_30s": g.get("best"), "generations_30s": g.get("generations")}
    sample = (f"{procs} processes x {'genopt.run()' if tb['kind'] == 'reference' else 'oracle port'}"
              f" (P=8, T=128, C2 + tsp-delta), generations {args.warmup + 1}-"
              f"{args.warmup + args.steps} timed")
    out = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "move evals/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tb["wall_s"] / max(1, args.steps),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded 26x17 lattice, permuted labels, TSPLIB nint)",
        "config": {"workload": "C2 pcb442-shaped lattice TSP n=442 + user tsp-delta ops",
                   "population_per_process": 8, "team_size": 128,
                   "generations_per_step": 1},
        "cpu_baseline": {"value": value, "unit": "move evals/s", "cores": procs,
                         "kind": tb["kind"], "cpu_model": R.cpu_model(), "sample": sample},
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
    ap.add_argument("--cpu-gens", type=int, default=2)
    ap.add_argument("--cpu-warm-gens", type=int, default=2)
    ap.add_argument("--other-gap-seconds", type=float, default=30.0,
                    help="wall-clock budget of the other shapes' gap runs (0 = skip)")
    ap.add_argument("--only", default="", help="comma list of other shapes to measure")
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
