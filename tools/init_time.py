import time, sys
sys.path.insert(0, "/root/repo")
import paper_2603_19163_b200 as G
from paper_2603_19163_b200 import instances as I
d, opt = I.tsp_lattice()
prob = G.builtin_problem("tsp", G.InstanceData(distance_matrix=d))
for rep, dev_init in ((0, False), (1, False), (2, True), (3, True)):
    t = time.perf_counter()
    dr = G.DeviceRun(prob, G.EngineConfig(custom_operators=G.tsp_delta_operators(),
                                          device_init=dev_init), 42)
    t1 = time.perf_counter()
    print(f"device_init={dev_init}: DeviceRun init {t1 - t:.3f} s (jit {dr.jit_seconds:.3f} s), P={dr.pop_size}")
    dr.close()
