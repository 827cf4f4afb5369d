"""Throughput vs teams per CTA for the JIT TSP kernel (register budget
GO_EVOLVE_MAX_THREADS): python tools/occupancy_probe.py C1|C2 E"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_19163_b200 as G  # noqa: E402
from paper_2603_19163_b200 import instances as I  # noqa: E402

name, E = sys.argv[1], int(sys.argv[2])
d = I.tsp_random(51, 51) if name == "C1" else I.tsp_lattice()[0]
prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=d))
dr = G.DeviceRun(prob, G.EngineConfig(seed=42, teams_per_cta=E, population=148 * E,
                                      custom_operators=G.tsp_delta_operators()), 42)
done = 20
dr.run(done, None)
ms = 0.0
for _ in range(5):
    done += 10
    ms += dr.run(done, None).device_ms
evals = dr.pop_size * 128 * 50
print(f"{name} E={E} max_threads={os.environ.get('GO_EVOLVE_MAX_THREADS', '512')} "
      f"P={dr.pop_size} teams/SM={dr.teams_per_sm}: {evals / (ms / 1e3) / 1e6:.1f} M evals/s")
dr.close()
