"""Phase timeline of the scan kernels (debug tracing via iir_debug_trace).

    python tools/trace_phases.py [--workload c2] [--reps 3]

Prints, per kernel, percentiles over tiles of each phase's start time relative
to the kernel's first tile start (microseconds)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2511_14390_b200 import _binding as B  # noqa: E402

PH_F = ["start", "local", "scan", "carry", "emit", "store", "-", "-"]
PH_B = ["start", "local", "scan", "carry", "emit", "store", "-", "-"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    w = dict(bench.WORKLOADS[a.workload], key=a.workload)
    prob = bench.Problem(w, 0, 1, 2)
    s = torch.cuda.Stream()
    ntot = w["batch"] * ((w["length"] + 4095) // 4096)
    buf = torch.zeros(ntot * 8, dtype=torch.int64, device="cuda")
    for rep in range(a.reps):
        with torch.cuda.stream(s):
            prob.step(0, s)
        torch.cuda.synchronize()
    for kern in ("fwd", "bwd"):
        buf.zero_()
        B.iir_debug_trace(buf)
        st = prob.sets[0]
        with torch.cuda.stream(s):
            if kern == "fwd":
                B.iir_forward(prob.desc, prob.b, prob.a, st["x"], prob.zi, st["y"], prob.zf, prob.tape, prob.tb,
                              prob.ws, prob.wb, s)
            else:
                B.iir_debug_trace(None)
                B.iir_forward(prob.desc, prob.b, prob.a, st["x"], prob.zi, st["y"], prob.zf, prob.tape, prob.tb,
                              prob.ws, prob.wb, s)
                B.iir_debug_trace(buf)
                B.iir_backward(prob.desc, st["gy"], prob.gzf, prob.b, prob.a, st["x"], st["y"], prob.zi, prob.tape,
                               prob.tb, st["gx"], prob.gb, prob.ga, prob.gzi, prob.ws, prob.wb, s)
        torch.cuda.synchronize()
        B.iir_debug_trace(None)
        t = buf.view(ntot, 8).cpu().numpy().astype(np.float64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        names = PH_F if kern == "fwd" else PH_B
        print(f"== {kern} ({ntot} tiles), us relative to first tile start; columns p0 p10 p50 p90 p100")
        for k, nm in enumerate(names[:6]):
            col = rel[:, k]
            col = col[t[:, k] > 0]
            if nm == "-" or col.size == 0:
                continue
            q = np.percentile(col, [0, 10, 50, 90, 100])
            print(f"   {nm:8s} " + " ".join(f"{v:8.2f}" for v in q))
        d = np.diff(rel, axis=1)
        print("   phase durations (median us): " + ", ".join(
            f"{names[k]}->{names[k + 1]} {np.median(d[:, k]):.2f}" for k in range(5)))


if __name__ == "__main__":
    main()
