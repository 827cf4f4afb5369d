"""Aggregates an ncu source page (--page source --csv --print-source cuda,sass)
by CUDA source line: warp-stall samples (all / by reason), instructions.

    ncu -i prof.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    fname = None
    header = None
    agg = defaultdict(lambda: defaultdict(float))
    src = {}
    total = 0.0
    for row in csv.reader(open(path)):
        if not row:
            continue
        if row[0] == "File Path":
            fname = row[1].split("/")[-1]
            continue
        if row[0] == "Function Name":
            continue
        if row[0] == "Line No":
            header = row
            continue
        if header is None or row[0] == "":
            continue  # SASS rows: the line row already carries the totals
        d = dict(zip(header, row))
        key = (fname, int(row[0]))
        src[key] = row[1][:70]
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k or k in (
                    "Warp Stall Sampling (All Samples)", "Instructions Executed"):
                try:
                    agg[key][k] += float(v)
                except ValueError:
                    pass
        total += agg[key]["Warp Stall Sampling (All Samples)"] * 0  # noqa
    tot = sum(a["Warp Stall Sampling (All Samples)"] for a in agg.values())
    by_file = defaultdict(float)
    for (f, _), a in agg.items():
        by_file[f] += a["Warp Stall Sampling (All Samples)"]
    print(f"total samples {tot:.0f}")
    for f, v in sorted(by_file.items(), key=lambda x: -x[1]):
        print(f"  {v / tot * 100:5.1f}%  {f}")
    rows = sorted(agg.items(), key=lambda x: -x[1]["Warp Stall Sampling (All Samples)"])[:top]
    for (f, ln), a in rows:
        s = a["Warp Stall Sampling (All Samples)"]
        reasons = sorted(((k[6:], v) for k, v in a.items() if k.startswith("stall_")),
                         key=lambda x: -x[1])[:3]
        rs = " ".join(f"{k}:{v / max(s, 1) * 100:.0f}%" for k, v in reasons if v > 0)
        print(f"{s / tot * 100:5.1f}% {f}:{ln:<5} inst={a['Instructions Executed']:.0f}  {rs}  | {src[(f, ln)]}")


if __name__ == "__main__":
    main()
