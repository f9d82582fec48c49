"""Summarise an .ncu-rep (raw page) into one block per launch: duration, DRAM
bytes and throughput, L2 (lts) throughput, issue activity, occupancy, top
warp-stall reasons.  Usage: python scripts/ncu_summary.py <report.ncu-rep>"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "dram_rd"),
    ("dram__bytes_write.sum", "dram_wr"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "l2%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
    ("sm__inst_executed.avg.per_cycle_active", "ipc"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__occupancy_limit_registers", "occ_lim_regs"),
    ("launch__occupancy_limit_shared_mem", "occ_lim_smem"),
    ("l1tex__t_sector_hit_rate.pct", "l1hit%"),
    ("lts__t_sector_hit_rate.pct", "l2hit%"),
    ("sm__cycles_elapsed.avg.per_second", "sm_hz"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print(f"== {d.get('ID')} {d.get('Kernel Name', '')[:90]}")
        parts = []
        for k, short in KEYS:
            if k in d:
                parts.append(f"{short}={d[k]}{u.get(k, '')}")
        print("   " + "  ".join(parts))
        stalls = [(k, d[k]) for k in hdr if k.startswith("smsp__average_warp_latency_issue_stalled_") or
                  (k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"))]
        vals = []
        for k, v in stalls:
            try:
                vals.append((float(v.replace(",", "")), k))
            except ValueError:
                pass
        vals.sort(reverse=True)
        print("   stalls: " + ", ".join(f"{k.split('stalled_')[-1]}={v:g}" for v, k in vals[:7]))


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
