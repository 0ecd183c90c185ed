"""Stall samples of one kernel of an ncu report, grouped by SASS opcode
(ncu -i REPORT --page source --print-source sass).  usage: REPORT KERNEL_REGEX"""
import csv
import io
import subprocess
import sys
from collections import Counter

rep, kern = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr = r[1]
rows = [x for x in r[2:] if len(x) == len(hdr)]
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_e = hdr.index("Instructions Executed")
num = lambda v: int(v) if v.strip().isdigit() else 0
tot = sum(num(x[i_s]) for x in rows)
op, ex = Counter(), Counter()
for x in rows:
    t = x[1].split()
    if not t:
        continue
    o = t[1] if t[0].startswith("@") else t[0]
    op[o.split(".")[0]] += num(x[i_s])
    ex[o.split(".")[0]] += num(x[i_e])
print(f"samples {tot}, sass lines {len(rows)}, warp instructions {sum(ex.values())}")
print("| opcode | stall samples | share | warp instr executed |")
print("|---|---|---|---|")
for k, v in op.most_common(30):
    print(f"| {k} | {v} | {v / max(tot, 1):.1%} | {ex[k]} |")
