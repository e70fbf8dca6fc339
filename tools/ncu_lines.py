"""Per-CUDA-source-line instruction and stall shares of one kernel in an ncu report
(cuda,sass source view).   python tools/ncu_lines.py REP KERNEL_REGEX [TOP]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kre}",
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
agg = defaultdict(lambda: [0.0, 0.0, ""])
fname = ""
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    try:
        st = float(r[4] or 0)
        ie = float(r[7] or 0)
    except ValueError:
        continue
    a = agg[(fname, ln)]
    a[0] += ie
    a[1] += st
    if r[1].strip():
        a[2] = r[1].strip()[:90]
ti = sum(v[0] for v in agg.values()) or 1
ts = sum(v[1] for v in agg.values()) or 1
print(f"total warp instructions {ti:.0f}, stall samples {ts:.0f}")
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{v[0] / ti * 100:5.1f}% instr {v[1] / ts * 100:5.1f}% stall  {f}:{ln}  {v[2]}")
print("-- by stall")
for (f, ln), v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"{v[0] / ti * 100:5.1f}% instr {v[1] / ts * 100:5.1f}% stall  {f}:{ln}  {v[2]}")
