"""Diagnostic: per-phase clock64 breakdown of the evolve kernel (GO_PHASE_TIMING)."""
import ctypes as C, os, sys
os.environ["GO_JIT_DEFINE"] = "GO_PHASE_TIMING=1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2603_19163_b200 as G
from paper_2603_19163_b200 import _native as N, instances as I
d, opt = I.tsp_lattice()
prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=d))
dr = G.DeviceRun(prob, G.EngineConfig(custom_operators=G.tsp_delta_operators()), 42)
for chunk in (50, 300):
    dr.run(chunk, None)
    out = (C.c_int64 * 16)()
    N.check(dr.lib.go_engine_debug_counters(dr.engine, out, 16))
    v = np.array(list(out), dtype=np.float64)
    names = ["-", "s0 rank", "s0 order", "s0 exec", "s0 coop", "s1 rank", "s1 order", "s1 exec", "s1 coop",
             "s2 rank", "s2 order", "s2 exec", "s2 coop", "argmin", "decide+apply+rec",
             "deferred (all steps)"]
    tot = v.sum()
    print(f"after {chunk} gens: total {tot:.3e} cycles")
    for nm, x in zip(names, v):
        if x: print(f"  {nm:18s} {x/tot*100:5.1f}%")
    w, kw = dr.weights()
    print("  weights", np.round(w, 3), "k", np.round(kw, 3))
