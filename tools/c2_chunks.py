"""Runs a few evolve chunks of one BASELINE shape (default C2 + tsp-delta, the
bench configuration) through DeviceRun — a short command for ncu:

    ncu --set full -k regex:go_evolve -s 5 -c 1 -o prof python tools/c2_chunks.py [C2|C3|C4|C5a|C5b|C1] [chunks]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2603_19163_b200 as G  # noqa: E402
from paper_2603_19163_b200 import instances as I  # noqa: E402


def make(name):
    if name == "C2":
        import os
        d, _ = I.tsp_lattice()
        coop = os.environ.get("GO_DEMO_LOOPS", "0") != "1"  # per-lane loop snippets when set
        return (G.builtin_problem("tsp", G.InstanceData(distance_matrix=d)),
                G.tsp_delta_operators(cooperative=coop))
    from tools.op_cost import problems  # noqa: E402
    return problems()[name](), ()


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    prob, ops = make(name)
    dr = G.DeviceRun(prob, G.EngineConfig(seed=42, custom_operators=ops), 42)
    done = 0
    for _ in range(chunks):
        done += 10
        st = dr.run(done, None)
        print(f"{name} chunk -> gen {done}: {st.device_ms:.2f} ms", flush=True)
    dr.close()


if __name__ == "__main__":
    main()
