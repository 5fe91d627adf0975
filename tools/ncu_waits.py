"""Per-barrier wait retries and per-region stall shares from an ncu report's
SASS page (which pipeline role is waiting on which mbarrier).
Usage: python tools/ncu_waits.py report.ncu-rep"""
import csv
import io
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
i_src, i_s, i_ex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
tot = sum(float(r[i_s] or 0) for r in data) or 1.0
waits = defaultdict(float)
for r in data:
    if "TRYWAIT" in r[i_src]:
        inner = r[i_src].split("[")[1].split("]")[0]
        bar = inner.split("+")[-1] if "+0x" in inner else "0x0(" + inner + ")"
        waits[bar] += float(r[i_ex] or 0)
print("mbarrier try_wait executions by barrier offset:")
for k, v in sorted(waits.items(), key=lambda x: -x[1]):
    print(f"  {k:>8s} {v:14.0f}")
bins = defaultdict(float)
for r in data:
    a = int(r[0], 16) & 0xfffff
    bins[a // 0x1000] += float(r[i_s] or 0)
print("stall samples by 4 KB code region:")
for k in sorted(bins):
    if bins[k] / tot > 0.02:
        print(f"  {k * 0x1000:#x} {100 * bins[k] / tot:5.1f}%")
