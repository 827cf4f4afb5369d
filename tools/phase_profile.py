"""Diagnostic: per-phase clock64 breakdown of the C2 evolve kernel and the mean
duration of each deferred whole-row operator (GO_PHASE_TIMING build)."""
import ctypes as C
import os
import sys

os.environ["GO_JIT_DEFINE"] = "GO_PHASE_TIMING=1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2603_19163_b200 as G  # noqa: E402
from paper_2603_19163_b200 import _native as N, instances as I  # noqa: E402

d, opt = I.tsp_lattice()
prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=d))
dr = G.DeviceRun(prob, G.EngineConfig(custom_operators=G.tsp_delta_operators()), 42)
names = ["-", "s0 rank", "s0 order", "s0 exec", "s0 coop", "s1 rank", "s1 order", "s1 exec",
         "s1 coop", "s2 rank", "s2 order", "s2 exec", "s2 coop", "argmin", "decide+apply+rec",
         "deferred (all steps)"]
prev = np.zeros(32)
for chunk in (50, 300):
    dr.run(chunk, None)
    out = (C.c_int64 * 32)()
    N.check(dr.lib.go_engine_debug_counters(dr.engine, out, 32))
    allv = np.array(list(out), dtype=np.float64)
    v = allv - prev
    prev = allv
    tot = v[:16].sum()
    print(f"up to generation {chunk}: team-thread total {tot:.3e} cycles "
          f"({tot / dr.pop_size / (chunk if chunk == 50 else 250):.0f} per team-generation)")
    for nm, x in zip(names, v[:16]):
        if x:
            print(f"  {nm:18s} {x / tot * 100:5.1f}%")
    for label, b in (("OX", 16), ("shuffles", 18), ("guided rebuild", 20)):
        if v[b + 1]:
            print(f"  {label:15s} {v[b + 1]:9.0f} applications, mean {v[b] / v[b + 1]:9.0f} cycles")
    if v[29]:
        print(f"  crossover mates: {v[29]:.0f} picks, {v[28]:.0f} waited "
              f"({v[28] / v[29] * 100:.1f} %), mean wait {v[27] / max(v[28], 1):.0f} cycles, "
              f"{v[27] / v[29]:.0f} cycles per pick")
    if v[17]:
        print(f"  OX parts (mean cycles): staging + kept slice {v[30] / v[17]:.0f}, "
              f"fill + length {v[31] / v[17]:.0f}")
    if v[26]:
        print("  lane execution per step, by warp index (mean cycles):",
              [int(v[22 + i] / v[26]) for i in range(4)])
    w, kw = dr.weights()
    print("  weights", np.round(w, 3), "k", np.round(kw, 3))
