"""Top CUDA source lines of one kernel in an .ncu-rep, by executed warp
instructions and warp-stall samples (aggregated from the cuda,sass view).
Usage: python scripts/ncu_lines.py rep.ncu-rep kernel_regex [n]"""
import csv
import io
import os
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass", "--launch-count", "1"], capture_output=True, text=True).stdout
agg = {}
fname = "?"
cur = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0]:  # a CUDA source line
        cur = (fname, r[0], r[1].strip()[:100])
        continue
    if cur is None or len(r) < 8 or r[2] in ("...", "-"):
        continue
    try:
        stall = int(r[4])
        inst = int(r[7])
    except ValueError:
        continue
    a = agg.setdefault(cur, [0, 0])
    a[0] += inst
    a[1] += stall
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {ti}, stall samples {ts}")
for (f, ln, src), (i, s) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*i/ti:5.1f}% inst {100*s/ts:5.1f}% stall  {f}:{ln}: {src}")
