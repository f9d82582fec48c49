"""Write the closing-pass summaries under profiles/ from gpurun_out/r02c_*
(bench line, launch list, traffic of the dominant kernels, ncu summaries,
sanitizer tails).  Dev-container helper: python scripts/summarize_r02c.py"""
import collections
import csv
import glob
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return [dict(zip(r[0], row)) for row in r[2:]]


# bench line
line = open(os.path.join(G, "r02c_bench.txt")).read().strip().splitlines()[-1]
json.loads(line)
open(os.path.join(P, "r02_bench.json"), "w").write(line + "\n")

# launch list
rows = list(csv.reader(open(os.path.join(G, "r02c_bench_launches.csv"))))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if not hdr or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    k = d["Kernel Name"]
    if "pfr::" not in k or "probe" in k:
        continue
    a = agg.setdefault(k, collections.defaultdict(float))
    a[d["Metric Name"]] += float(d["Metric Value"].replace(",", ""))
    if d["Metric Name"] == "gpu__time_duration.sum":
        a["n"] += 1
reps = 9
tot = sum(a["gpu__time_duration.sum"] for a in agg.values()) / reps / 1e3
lines = ["# round 2 closing pass (scripts/gpu_r02c_final.sh): ncu launch list of `python bench.py --steps 2 "
         "--warmup 1 --no-targets --no-cpu-baseline`",
         "# (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none; "
         "cold caches, serialised launches).  Every delivery ran 9 times over the bench legs; per step = sum / 9.",
         "# Only this library's kernels (torch's flush / spin / fill kernels and the gather probe excluded).",
         "# Share = the kernel's part of the step's library kernel time; compare with per_delivery_ms of the bench line.",
         f"# total library kernel time per step (serialised): {tot:.1f} us"]
for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
    us = a["gpu__time_duration.sum"] / reps / 1e3
    mb = (a["dram__bytes_read.sum"] + a["dram__bytes_write.sum"]) / a["n"] / 1e6
    lines.append(f"  {us:8.1f} us/step {100 * us / tot:5.1f}%  launches/step {a['n'] / reps:4.1f}  "
                 f"dram {mb:8.2f} MB/launch  {k[:150]}")
open(os.path.join(P, "r02c_bench_launches.txt"), "w").write("\n".join(lines) + "\n")

# traffic of the rejection kernels
tp = os.path.join(P, "r02_traffic.json")
t = json.load(open(tp))
for dt in ("f32", "f64"):
    rs = raw(os.path.join(G, f"r02c_rejection_{dt}.ncu-rep"))
    main = [x for x in rs if "k_rejection_philox" in x["Kernel Name"]][0]
    tab = [x for x in rs if "k_rej_table" in x["Kernel Name"]][0]
    b = lambda x: (float(x["dram__bytes_read.sum"]) + float(x["dram__bytes_write.sum"])) * 1e6  # noqa: E731
    t[f"rejection/{dt}"] = {"kernel": main["Kernel Name"][:80], "bytes": round(b(main)),
                            "table_kernel_bytes": round(b(tab)),
                            "source": f"r02c_rejection_{dt}.ncu-rep (--set full, closing pass)"}
json.dump(t, open(tp, "w"), indent=1)

# ncu summaries
want = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio"]
out = ["# round 2 closing pass: ncu --set full --clock-control none (cold caches), scripts/gpu_r02c_final.sh",
       "# rejection 2^20 (sigma=1, sup=max w) f32 then f64: k_rej_table + k_rejection_philox; own-stream "
       "multinomial 2^20 f32: weight scan + k_mn_tilesum / k_mn_tileprefix / k_mn_merge"]
for f in ("r02c_rejection_f32", "r02c_rejection_f64", "r02c_multinomial"):
    for x in raw(os.path.join(G, f + ".ncu-rep")):
        out.append(f"== {f} {x['Kernel Name'][:90]}")
        out += [f"    {w} {x[w]}" for w in want if w in x]
out.append("# per-line instruction / stall shares of the rejection kernel, f32 (scripts/ncu_lines.py)")
out.append(subprocess.run(["python", os.path.join(ROOT, "scripts", "ncu_lines.py"),
                           os.path.join(G, "r02c_rejection_f32.ncu-rep"), "k_rejection_philox", "16"],
                          capture_output=True, text=True).stdout)
open(os.path.join(P, "r02c_full.txt"), "w").write("\n".join(out) + "\n")

# sanitizers
san = ["# round 2 closing pass sanitizers (scripts/gpu_r02c_final.sh)"]
for f in sorted(glob.glob(os.path.join(G, "r02c_sanitize_*"))):
    san.append(f"== {os.path.basename(f)}")
    san += open(f).read().strip().splitlines()[-2:]
open(os.path.join(P, "r02c_sanitizers.txt"), "w").write("\n".join(san) + "\n")
print("\n".join(lines[4:14]))
