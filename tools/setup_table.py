"""Setup kernels' device time and DRAM traffic (achieved HBM GB/s) from an ncu --csv metrics log of
tools/prof_setup.py (gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum).

    python tools/setup_table.py gpurun_out/setup_c3.csv [hbm_gbs]
"""
import collections
import csv
import io
import sys


def kernel_name(k):
    base = k.split("(")[0].replace("<unnamed>", "").replace("void ", "")
    depth, out = 0, ""
    for ch in base:  # drop template arguments
        if ch == "<":
            depth += 1
        elif ch == ">":
            depth -= 1
        elif depth == 0:
            out += ch
    return out.split("::")[-1]


def main(path, peak=6536.4):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    h, data = rows[0], [r for r in rows[1:] if r[0] != "ID"]
    ik, im, iv, iid = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in data:
        try:
            per[(int(r[iid]), r[ik])][r[im]] = float(r[iv].replace(",", ""))
        except ValueError:
            pass
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, k), m in per.items():
        a = agg[kernel_name(k)]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0) / 1e3
        a[2] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
    tot = sum(a[1] for a in agg.values())
    print(f"| kernel | launches | device time (us) | DRAM bytes | achieved GB/s | of {peak:.0f} GB/s | share of time |")
    print("|---|---|---|---|---|---|---|")
    for n, a in sorted(agg.items(), key=lambda x: -x[1][1])[:16]:
        gbs = a[2] / (a[1] * 1e-6) / 1e9 if a[1] else 0.0
        print(f"| {n} | {a[0]} | {a[1]:.1f} | {a[2] / 1e6:.1f} MB | {gbs:.0f} | {gbs / peak:.2f} | {a[1] / tot * 100:.1f} % |")
    b = sum(a[2] for a in agg.values())
    print(f"| **all setup kernels** | {sum(a[0] for a in agg.values())} | {tot:.1f} | {b / 1e6:.1f} MB | "
          f"{b / (tot * 1e-6) / 1e9:.0f} | {b / (tot * 1e-6) / 1e9 / peak:.2f} | 100 % |")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 6536.4)
