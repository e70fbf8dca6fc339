"""Kernel spans of one fwd + bwd step (debug tracing via iir_debug_trace), for
either LTI scan schedule, eager and captured in a CUDA graph; plus the phase
stamps of the three-phase carry scan (sequence 0).

    python tools/trace_3p.py [--workload c4] [--scan 3p]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2511_14390_b200 import _binding as B  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c4")
    ap.add_argument("--scan", default="3p")
    a = ap.parse_args()
    w = dict(bench.WORKLOADS[a.workload], key=a.workload, scan=a.scan)
    prob = bench.Problem(w, 0, 1, 2)
    s = torch.cuda.Stream()
    ts = 128 * (32 if w["dtype"] == "f32" else 16) * (2 if w["order"] >= 4 else 1)
    ntot = w["batch"] * ((w["length"] + ts - 1) // ts)
    buf = torch.zeros(ntot * 16 + 64, dtype=torch.int64, device="cuda")
    st = prob.sets[0]

    def step():
        B.iir_debug_trace(buf)
        B.iir_forward(prob.desc, prob.b, prob.a, st["x"], prob.zi, st["y"], prob.zf, prob.tape, prob.tb,
                      prob.ws, prob.wb, s)
        B.iir_backward(prob.desc, st["gy"], prob.gzf, prob.b, prob.a, st["x"], st["y"], prob.zi, prob.tape,
                       prob.tb, st["gx"], prob.gb, prob.ga, prob.gzi, prob.ws, prob.wb, s)
        B.iir_debug_trace(None)

    def reset():
        buf.zero_()
        buf[ntot * 16::2] = (1 << 63) - 1

    def report(tag):
        g = buf[ntot * 16:].cpu().numpy().astype(np.float64)
        t0 = g[0]
        names = {0: "prep", 8: "red_fwd", 10: "cscan_fwd", 2: "fwd", 12: "red_bwd", 14: "cscan_bwd", 4: "bwd"}
        parts = []
        for o in (0, 8, 10, 2, 12, 14, 4):
            if g[o] < 9e18 and g[o + 1] > 0:
                parts.append(f"{names[o]} [{(g[o] - t0) / 1e3:.2f}, {(g[o + 1] - t0) / 1e3:.2f}]")
        print(f"== {tag}: " + ", ".join(parts))
        for o, nm in ((16, "cscan_fwd"), (32, "cscan_bwd")):
            st_ = g[o:o + 7]
            if st_[0] > 0 and st_[0] < 9e18:
                print(f"   {nm} stamps (us from its entry): " +
                      " ".join(f"{(v - st_[0]) / 1e3:.2f}" for v in st_[1:]) +
                      "   [wait, x0, horner, warp+block, walk, end]")

    with torch.cuda.stream(s):
        for _ in range(3):
            reset()
            step()
    torch.cuda.synchronize()
    report("eager")
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        step()
    torch.cuda.synchronize()
    for _ in range(3):
        reset()
        gr.replay()
        torch.cuda.synchronize()
    report("graph")


if __name__ == "__main__":
    main()
