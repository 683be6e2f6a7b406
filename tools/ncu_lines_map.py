"""Stall samples of one kernel, per CUDA source region: ncu source page (SASS, absolute
addresses) + nvdisasm -g line info of the same cubin.

    python tools/ncu_lines_map.py report.ncu-rep all_lines.txt <mangled-kernel-substring> <source.cu>
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, lines_txt, ksub, srcf = sys.argv[1:5]
txt = open(lines_txt).read().split("\n")
start = [i for i, l in enumerate(txt) if l.strip().startswith(".section") and ".text." in l and ksub in l][0]
addr2line, cur = {}, None
for l in txt[start + 1:]:
    if l.strip().startswith(".section"):
        break
    m = re.search(r'File "([^"]+)", line (\d+)', l)
    if m and "//##" in l:
        cur = int(m.group(2)) if m.group(1).endswith(srcf.split("/")[-1]) else -2
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
    if m and cur is not None:
        addr2line[int(m.group(1), 16)] = cur
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, data = rows[1], rows[2:]
ia, iall = h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
addrs = [int(r[ia], 16) for r in data if r[ia].startswith("0x")]
base = min(addrs)
src = open(srcf).read().split("\n")
byline, tot = defaultdict(float), 0.0
for r in data:
    if not r[ia].startswith("0x"):
        continue
    v = float(r[iall] or 0)
    tot += v
    byline[addr2line.get(int(r[ia], 16) - base, -1)] += v
names = ["fstep", "fpair", "apply_fixed", "zrot", "stage1", "stage2", "stage3", "m2l_v4_kernel", "write_target",
         "finish_segment", "dev_sph_jn", "rsqrt_nr", "cp_async8", "cp_async_wait_all"]


def region(ln):
    if ln == -2:
        return "(other file)"
    if ln < 0 or ln > len(src):
        return "unknown"
    for k in range(ln - 1, max(0, ln - 150), -1):
        s = src[k]
        if s.startswith(("__device__", "__global__", "template", "void")) or "__forceinline__" in s:
            for nm in names:
                if re.search(r"\b" + nm + r"\s*\(", s):
                    return nm
    return "other"


agg = defaultdict(float)
for ln, v in byline.items():
    agg[region(ln)] += v
for k, v in sorted(agg.items(), key=lambda x: -x[1]):
    print(f"{k:18s} {v / tot * 100:5.1f}%")
print("top lines:")
for ln, v in sorted(byline.items(), key=lambda x: -x[1])[:25]:
    print(f"{ln:5d} {v / tot * 100:5.1f}%  {src[ln - 1].strip()[:100] if ln > 0 else ''}")
