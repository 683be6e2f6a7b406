"""Summarise an ncu --csv launch list (gpu__time_duration.sum per launch) by kernel.

    python tools/ncu_summary.py gpurun_out/launches.csv [--skip-setup]
"""
import collections
import csv
import re
import sys


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = []
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki]
        name = re.sub(r"\(.*$", "", name)
        name = name.replace("fmm::<unnamed>::", "").replace("void ", "")
        name = re.sub(r"^at::native::.*?(\w+kernel).*$", r"torch:\1", name)
        v = float(r[vi].replace(",", ""))
        v *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(r[ui], 1.0)
        out.append((name, v))
    return out


def main():
    path = sys.argv[1]
    L = load(path)
    agg = collections.OrderedDict()
    for n, v in L:
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(a[1] for a in agg.values())
    print(f"| kernel | launches | total us | share |\n|---|---|---|---|")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {n} | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    print(f"\ntotal {tot / 1e3:.2f} ms over {len(L)} launches")


if __name__ == "__main__":
    main()
