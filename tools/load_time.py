import sys, time
sys.path.insert(0, "/root/repo")
t = time.perf_counter()
from paper_2603_19163_b200 import build as B
print("needs_build", B.needs_build(), flush=True)
from paper_2603_19163_b200 import _native as N
t1 = time.perf_counter()
import os
os.environ["GO_AUTOBUILD"] = "0"
N.load()
t2 = time.perf_counter()
print(f"import {t1 - t:.2f}s load {t2 - t1:.2f}s", flush=True)
import ctypes as C
n = C.c_int()
t3 = time.perf_counter()
N.check(N._lib.go_device_count(C.byref(n)))
info = N.device_info(0)
t4 = time.perf_counter()
print(f"device query {t4 - t3:.2f}s", flush=True)
