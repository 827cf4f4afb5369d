"""Per-operator cost on the device: ms per 10-generation chunk for each BASELINE
shape with the full registry, then with one operator removed at a time.
    python tools/op_cost.py [config ...]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2603_19163_b200 as G  # noqa: E402
from paper_2603_19163_b200 import instances as I  # noqa: E402


def problems():
    vd = I.vrptw_solomon_like()
    f, dq = I.qap_random(100, 100)
    w, v, cap = I.knapsack_random(1000, 1000)
    d, _ = I.tsp_lattice()
    return {
        "C1": lambda: G.builtin_problem("tsp", G.InstanceData(distance_matrix=I.tsp_random(51, 51))),
        "C2": lambda: G.builtin_problem("tsp", G.InstanceData(distance_matrix=d)),
        "C3": lambda: G.builtin_problem("vrptw", G.InstanceData(
            distance_matrix=vd.dist, demands=vd.demands, capacity=vd.capacity,
            vehicles=vd.vehicles, ready_times=vd.ready, due_times=vd.due,
            service_times=vd.service)),
        "C4": lambda: G.builtin_problem("qap", G.InstanceData(flow_matrix=f, distance_matrix=dq)),
        "C5a": lambda: G.builtin_problem("jsp_int", G.InstanceData(jobs=I.jsp_random(20, 15, 2015))),
        "C5b": lambda: G.builtin_problem("knapsack", G.InstanceData(weights=w, values=v,
                                                                     capacity=cap)),
    }


def time_cfg(make, ops, steps=6, gps=10):
    prob = make()
    if ops is not None:
        prob.device_sequences = lambda: ops
    custom = G.tsp_delta_operators() if CUSTOM else ()
    aos = G.AosConfig(update_interval=10 ** 9) if FROZEN else G.AosConfig()
    dr = G.DeviceRun(prob, G.EngineConfig(seed=42, custom_operators=custom, aos=aos), 42)
    done = gps
    dr.run(done, None)
    ms = 0.0
    per = []
    for _ in range(steps):
        done += gps
        t = dr.run(done, None).device_ms
        per.append(round(t, 2))
        ms += t
    w, kw = dr.weights()
    w = {e.id: round(float(x), 4) for e, x in zip(dr.registry.entries, w)}
    dr.close()
    return ms / steps, (w, [round(float(x), 3) for x in kw], per)


CUSTOM = "--custom" in sys.argv
FROZEN = "--frozen" in sys.argv  # no AOS updates: the preset operator mix throughout


def main():
    sel = [a for a in sys.argv[1:] if not a.startswith("--")] or ["C1", "C2", "C3", "C4", "C5a", "C5b"]
    P = problems()
    for name in sel:
        make = P[name]
        full = make().device_sequences()
        t_full, w = time_cfg(make, None)
        print(f"{name}: full registry {t_full:.2f} ms/chunk  ops={full}", flush=True)
        print(f"   weights {w[0]} k {w[1]} per-chunk {w[2]}", flush=True)
        if "--full" in sys.argv:
            continue
        for op in full:
            rest = tuple(o for o in full if o != op)
            try:
                t, _ = time_cfg(make, rest)
                print(f"   without {op:>2}: {t:9.2f} ms/chunk", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"   without {op:>2}: error {e}", flush=True)


if __name__ == "__main__":
    main()
