"""Compiles the C2 evolve kernel (int16 triangle + tsp-delta user operators)
with NVRTC here (no GPU needed) and prints its registers / stack / spills
and SASS size — the check to run before spending GPU time.

    GO_EVOLVE_MAX_THREADS=384 python tools/jit_resources.py [layout]
"""
import ctypes as C
import glob
import os
import subprocess
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2603_19163_b200 import _native as N  # noqa: E402
from paper_2603_19163_b200.demo_ops import tsp_delta_operators  # noqa: E402


def main():
    layout = int(sys.argv[1]) if len(sys.argv) > 1 else 1  # 1 = DistI16Tri
    lib = N.load(require_device=False)
    ops = tsp_delta_operators()
    arr = (N.CustomOp * len(ops))()
    keep = []
    for i, op in enumerate(ops):
        name, body = op.name.encode(), op.cuda.encode()
        keep += [name, body]
        arr[i] = N.CustomOp(op.id, name, body)
    log = C.create_string_buffer(1 << 16)
    key = C.create_string_buffer(65)
    rc = lib.go_jit_compile(layout, arr, len(ops), log, len(log), key)
    if rc:
        print(log.value.decode()[-4000:])
        sys.exit(1)
    cache = os.environ.get("GO_JIT_CACHE") or os.path.expanduser("~/.cache/cugenopt")
    cubin = os.path.join(cache, key.value.decode() + ".cubin")
    out = subprocess.run(["cuobjdump", "--dump-resource-usage", cubin], capture_output=True,
                         text=True).stdout
    for line in out.splitlines():
        if "go_evolve" in line or "REG" in line:
            print(line.strip())
    sass = subprocess.run(["cuobjdump", "-sass", cubin], capture_output=True, text=True).stdout
    body = [ln for ln in sass.splitlines() if "/*" in ln and ";" in ln]
    print(f"SASS instructions (all kernels): {len(body)}; LDL {sum('LDL' in l for l in body)} "
          f"STL {sum('STL' in l for l in body)}")
    print(cubin)


if __name__ == "__main__":
    main()
