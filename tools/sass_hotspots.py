"""Source-line hot spots of one kernel from an ncu report (SASS page) and the
cubin's line table.

    python tools/sass_hotspots.py REPORT.ncu-rep KERNEL CUBIN [top]

Every SASS instruction's stall samples / executed instructions are attributed
to the innermost source line nvdisasm -g reports for its offset.
"""
import collections
import csv
import io
import re
import subprocess
import sys


def line_table(cubin, kernel):
    out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    sec = None
    cur = None
    table = {}
    for ln in out.splitlines():
        m = re.match(r"//-+ \.text\.(\S+)\s", ln)
        if m:
            sec = m.group(1)
            continue
        if sec != kernel:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            table[int(m.group(1), 16)] = cur
    return table


def main():
    rep, kernel, cubin = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "-k", kernel], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    ia, iss, ie = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), \
        hdr.index("Instructions Executed")
    data = [r for r in rows[hdr_i + 1:] if len(r) == len(hdr)]
    base = int(data[0][ia], 16)
    lt = line_table(cubin, kernel)
    stall = collections.Counter()
    inst = collections.Counter()
    for r in data:
        off = int(r[ia], 16) - base
        key = lt.get(off, "?")
        stall[key] += float(r[iss] or 0)
        inst[key] += float(r[ie] or 0)
    ts, ti = sum(stall.values()), sum(inst.values())
    print(f"{kernel}: {ts:.0f} stall samples, {ti:.3e} warp instructions")
    for key, v in stall.most_common(top):
        print(f"{100 * v / ts:6.2f}% samples {100 * inst[key] / ti:6.2f}% inst  {key}")


if __name__ == "__main__":
    main()
