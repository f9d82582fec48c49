"""Aggregate an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel.
Usage: python scripts/ncu_launch_table.py <launches.csv>"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = d["Kernel Name"][:60]
    a = agg.setdefault(k, collections.defaultdict(float))
    a[d["Metric Name"]] += float(d["Metric Value"].replace(",", ""))
    if d["Metric Name"] == "gpu__time_duration.sum":
        a["n"] += 1
for k, a in agg.items():
    n = a["n"]
    t = a["gpu__time_duration.sum"] / n
    gb = (a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)) / n / 1e9
    print(f"{k:60s} n={n:4.0f} avg={t / 1e3:9.1f} us  dram={gb:7.3f} GB/launch  {gb / max(t, 1e-9) * 1e9 / 1e3:7.0f} GB/s")
