"""Timing table (median device time per cell, microseconds) and RMSE aggregate
of a `bench run` CSV: python scripts/grid_tables.py <in.csv> <precision> <times.txt> <rmse.csv>"""
import collections
import csv
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1301_4019_b200.bench_grid import aggregate_rmse, read_records_csv, write_rmse_csv  # noqa: E402

src, prec, times_out, rmse_out = sys.argv[1:5]
rows = list(csv.DictReader(open(src)))
algs = sorted({r["algorithm"] for r in rows})
ys = sorted({float(r["y"]) for r in rows})
ns = sorted({int(r["N"]) for r in rows})
cell = collections.defaultdict(list)
for r in rows:
    if r["mse"] != "":
        cell[(r["algorithm"], int(r["N"]), float(r["y"]))].append(int(r["elapsed_ns"]) / 1e3)
out = [f"# `python -m paper_1301_4019_b200 bench run --n 2^10..2^20 --y 0..4:2 --reps 3 --precision {prec}` on one B200",
       "# (the reference's grid and CSV schema; elapsed = device time of resample + permute, median of 3 reps,",
       "# microseconds; status words read after the timed region)",
       "# the paper's timing surfaces (PAPER.md Figs. 3-4) are figures only; this is the B200 counterpart", ""]
for y in ys:
    out.append(f"## y = {y}")
    out.append(f"{'N':>9}" + "".join(f"{a[:14]:>16}" for a in algs))
    for n in ns:
        out.append(f"{n:>9}" + "".join(f"{statistics.median(cell[(a, n, y)]):16.1f}" if cell[(a, n, y)]
                                        else f"{'err':>16}" for a in algs))
    out.append("")
open(times_out, "w").write("\n".join(out))
write_rmse_csv(aggregate_rmse(read_records_csv(src)), rmse_out)
print("\n".join(out[:19]))
