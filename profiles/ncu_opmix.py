"""Instruction mix + top stall lines of one kernel in an ncu report (run here).

    python profiles/ncu_opmix.py report.ncu-rep <kernel regex> [launch index]
"""
import collections
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
idx = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}", "--launch-skip", idx,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
print(rows[0][1][:100])
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
ie = hdr.index("Instructions Executed")
si = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[ie]) for r in data if r[ie].isdigit())
ops = collections.Counter()
for r in data:
    if r[ie].isdigit():
        t = r[1].strip().split()
        op = t[1] if t[0].startswith("@") else t[0]
        ops[op.split(".")[0]] += int(r[ie])
print("total warp instructions", tot)
for k, v in ops.most_common(22):
    print(f"  {k:12s} {v:11d} {100 * v / tot:5.1f}%")
stot = sum(int(r[si]) for r in data if r[si].isdigit()) or 1
print("top stall lines:")
for i, r in sorted(enumerate(data), key=lambda ir: -int(ir[1][si]) if ir[1][si].isdigit() else 0)[:12]:
    print(f"  {100 * int(r[si]) / stot:5.1f}%  {i:5d} {r[1].strip()[:70]}")
