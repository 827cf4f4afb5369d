"""Static instruction footprint of one kernel, attributed to source functions.

    cuobjdump -xelf engine.sm_100a.cubin paper_2603_19163_b200/lib/libcugenopt.so
    nvdisasm -gi engine.sm_100a.cubin > eng.txt
    python tools/sass_attr.py eng.txt go_evolve_part [--callers]

Each SASS instruction is charged to the innermost source line of its inline
chain (nvdisasm -gi) and that line to the enclosing function definition
(a regex over the .cuh sources).  --callers charges it instead to the
outermost inline frame below the kernel body, i.e. which call site of the
kernel's own code pulled the instructions in.  Used to find what to move out
of line when the instruction cache hit rate is low."""
import re
import signal
import sys
from collections import Counter
from pathlib import Path

FILE_RE = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
INS_RE = re.compile(r"^\s+/\*[0-9a-f]{4,}\*/\s+\S")
DEF_RE = re.compile(r"^(?:template\s*<.*>\s*)?(?:static\s+)?(?:__device__|__global__|struct|inline)"
                    r"[^;{(]*?(\w+)\s*\(")
STRUCT_RE = re.compile(r"^\s*(?:struct|class)\s+(\w+)")


def func_map(path, cache={}):
    if path in cache:
        return cache[path]
    starts = []
    try:
        lines = Path(path).read_text().splitlines()
    except OSError:
        lines = []
    struct = None
    for i, ln in enumerate(lines, 1):
        m = STRUCT_RE.match(ln)
        if m and not ln.rstrip().endswith(";"):
            struct = m.group(1)
        if ln.startswith("}"):
            struct = None
        m = re.search(r"__device__[^;]*?(\w+(?:\[\])?)\s*\(", ln) or (ln.startswith("__global__") and
                                                             re.search(r"(\w+)\s*\(", ln))
        if m:
            name = m.group(1)
            starts.append((i, f"{struct}::{name}" if (struct and ln.startswith("  ")) else name))
    cache[path] = starts
    return starts


def func_of(path, line):
    best = "?"
    for s, name in func_map(path):
        if s <= line:
            best = name
        else:
            break
    return f"{Path(path).name}:{best}"


def main():
    signal.signal(signal.SIGPIPE, signal.SIG_DFL)
    txt, kern = sys.argv[1], sys.argv[2]
    callers = "--callers" in sys.argv
    lines = Path(txt).read_text().splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.strip() == f".text.{kern}:")
    chain, pending, by_fn, by_file = [], [], Counter(), Counter()
    total = 0
    for ln in lines[start + 1:]:
        if ln.startswith(".text.") or ln.startswith("\t.section"):
            break
        m = FILE_RE.search(ln)
        if m:
            pending.append((m.group(1), int(m.group(2))))
            continue
        if INS_RE.match(ln):
            if pending:
                chain, pending = pending, []
            if not chain:
                continue
            total += 1
            if callers:
                # frames innermost .. outermost; the kernel body frame is the last
                frame = chain[-2] if len(chain) >= 2 else chain[-1]
                key = f"{Path(frame[0]).name}:{frame[1]} ({func_of(*frame)})"
            else:
                key = func_of(*chain[0])
            by_fn[key] += 1
            by_file[Path(chain[0][0]).name] += 1
    print(f"{kern}: {total} instructions")
    for f, c in by_file.most_common():
        print(f"  {c:7d}  {f}")
    print()
    for f, c in by_fn.most_common(40):
        print(f"  {c:7d}  {f}")


if __name__ == "__main__":
    main()
