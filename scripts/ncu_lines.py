"""Per-source-line share of executed instructions and stall samples of one
kernel in an ncu report: python scripts/ncu_lines.py REPORT KERNEL_REGEX [TOP]"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30


def page(kind):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kern,
                          "--launch-count", "1", "--print-source", kind], capture_output=True, text=True).stdout
    return list(csv.reader(out.splitlines()))


addr2line, f, line = {}, None, None
for r in page("cuda,sass"):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) >= 4 and r[0] not in ("", "Line No", "Function Name"):
        line = (f, r[0], r[1])
    if len(r) >= 4 and r[2].startswith("0x"):
        addr2line[r[2]] = line
s = page("sass")
h = s[1]
ie, sp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
by, st, ops = collections.Counter(), collections.Counter(), collections.Counter()
for r in s[2:]:
    if len(r) <= ie or not r[0].startswith("0x"):
        continue
    n = int(r[ie] or 0)
    k = addr2line.get(r[0], ("?", "?", "?"))
    by[k] += n
    st[k] += int(r[sp] or 0)
    ops[r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]] += n
tot, tots = sum(by.values()), max(1, sum(st.values()))
print(f"warp instructions {tot}, stall samples {tots}")
for k, v in by.most_common(top):
    print(f"{100 * v / tot:5.1f}% instr {100 * st[k] / tots:5.1f}% stall  {k[0]}:{k[1]} {k[2][:90]}")
print("opcodes:", ", ".join(f"{o} {100 * v / tot:.1f}%" for o, v in ops.most_common(16)))
