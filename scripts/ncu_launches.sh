#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_targets.py ${WHICH:-all} 2 > gpurun_out/ncu_stdout.txt 2>&1
echo "ncu rc=$?"
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hdr = None
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr = i; break
h = rows[hdr]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
idi = h.index("ID")
agg = {}
for r in rows[hdr+1:]:
    if len(r) < len(h): continue
    agg.setdefault((int(r[idi]), r[ki][:60]), {})[r[mi]] = r[vi]
for (i, k), m in sorted(agg.items()):
    print(i, k, m.get("gpu__time_duration.sum"), m.get("dram__bytes_read.sum"), m.get("dram__bytes_write.sum"))
PY
