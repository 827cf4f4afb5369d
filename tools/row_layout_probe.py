"""Diagnostic: throughput of a row shape under each lane-row / instance placement
(GO_ROW_LAYOUT=10..13 forces the first layout choose_row may take):

    for L in 10 11 12 13; do GO_ROW_LAYOUT=$L python tools/row_layout_probe.py C5b; done
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2603_19163_b200 as G  # noqa: E402
from tools.op_cost import problems  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C5b"
    chunks = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    prob = problems()[name]()
    dr = G.DeviceRun(prob, G.EngineConfig(seed=42), 42)
    done, ms = 0, []
    for _ in range(chunks):
        done += 10
        ms.append(dr.run(done, None).device_ms)
    m = sum(ms[-3:]) / 3
    P, T = dr.pop_size, dr.config.team_size
    print(f"{name} layout {os.environ.get('GO_ROW_LAYOUT', 'auto')}: P={P} {m:.2f} ms/chunk "
          f"{P * T * 10 / m / 1e3:.2f} M evals/s")
    dr.close()


if __name__ == "__main__":
    main()
