"""Diagnostic: C3 (R101 fixture) runs — best objective / penalty / vehicles
after a wall-clock budget, for several seeds."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2603_19163_b200 as G  # noqa: E402
from paper_2603_19163_b200 import instances as I  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
kind, inst, _ = I.baseline_instances()["C3"]
prob = G.builtin_problem(kind, inst)
for seed in (1, 2):
    r = G.run(prob, G.EngineConfig(seed=seed, device_init=True, time_limit_seconds=secs,
                                   max_generations=10 ** 9))
    print(seed, r.objectives, r.penalty, r.generations_completed,
          r.config["population_effective"], flush=True)
