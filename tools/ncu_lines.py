"""Aggregate an ncu source page (cuda,sass correlation) by CUDA source line.

    ncu -i X.ncu-rep --page source --csv --print-source cuda,sass > src.csv
    python tools/ncu_lines.py src.csv [top]

Prints the top lines by warp-stall samples with their share of executed instructions and
excess shared-memory wavefronts (bank conflicts).
"""
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    agg = {}
    fname = "?"
    hdr = None
    for r in csv.reader(open(path)):
        if len(r) >= 2 and r[0] == "File Path":
            fname = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr) or not r[0].strip():
            continue
        d = dict(zip(hdr[4:], r[4:]))
        key = (fname, int(r[0]), r[1][:80])

        def f(k):
            try:
                return float(d.get(k, "0") or 0)
            except ValueError:
                return 0.0

        a = agg.setdefault(key, [0.0, 0.0, 0.0])
        a[0] += f("Warp Stall Sampling (All Samples)")
        a[1] += f("Instructions Executed")
        a[2] += f("L1 Wavefronts Shared Excessive")
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    for k, v in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
        print(f"{100 * v[0] / ts:5.1f}% stall {100 * v[1] / ti:5.1f}% inst  excess_wf={v[2]:.3g}  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main()
