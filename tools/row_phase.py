"""Diagnostic: per-phase clock64 breakdown of a row evolve kernel (C1, C3, C4,
C5a, C5b) from a GO_ROW_TIMING build of the library, e.g.

    git worktree add ab_kernels/rowtime HEAD
    (cd ab_kernels/rowtime && GO_NVCC_DEFINES=-DGO_ROW_TIMING python -c \\
        "import __graft_entry__ as g; g.build()")
    (cd ab_kernels/rowtime && python tools/row_phase.py C3)       # on the GPU
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2603_19163_b200 as G  # noqa: E402
from paper_2603_19163_b200 import _native as N  # noqa: E402
from tools.op_cost import problems  # noqa: E402

PHASES = ["copy + draws", "regroup", "lane execution (+ barrier wait)", "deferred uniform X",
          "deferred guided rebuild", "evaluation", "acceptance + records"]
KINDS = ["swap", "insert", "reverse", "or_opt", "three_opt", "flip", "seg_flip", "random_reset",
         "seg_reset", "row_swap", "row_split", "row_merge", "ox", "uniform_x", "seg_shuffle",
         "scatter_shuffle"]


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C3"
    prob = problems()[name]()
    dr = G.DeviceRun(prob, G.EngineConfig(seed=42), 42)
    prev = np.zeros(32)
    for upto in (20, 70):
        dr.run(upto, None)
        out = (C.c_int64 * 32)()
        N.check(dr.lib.go_engine_debug_counters(dr.engine, out, 32))
        allv = np.array([int(x) & ((1 << 64) - 1) for x in out], dtype=np.float64)
        raw = [int(x) & ((1 << 64) - 1) for x in out]
        v = allv - prev
        prev = allv
        gens = 20 if upto == 20 else 50
        tot = v[:7].sum()
        print(f"{name} up to generation {upto}: {tot / dr.pop_size / gens:.0f} cycles per "
              f"team-generation (population {dr.pop_size})")
        for nm, x in zip(PHASES, v[:7]):
            print(f"  {nm:34s} {x / tot * 100:5.1f}%")
        print("  lane execution by warp (cycles per team-generation):",
              [int(v[8 + i] / dr.pop_size / gens) for i in range(4)])
        if upto == 70:
            for k, nm in enumerate(KINDS):
                r = raw[12 + k]
                cnt, cyc = r >> 40, r & ((1 << 40) - 1)
                if cnt:
                    print(f"  {nm:16s} {cnt:9d} applications (all chunks), mean {cyc / cnt:8.0f} cycles")
    dr.close()


if __name__ == "__main__":
    main()
