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

PH_F = ["start", "local", "scan", "carry", "emit", "store", "lvl0", "lvl1"]
PH_B = ["start", "local", "scan", "carry", "emit", "store", "lvl0", "lvl1"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    w = dict(bench.WORKLOADS[a.workload], key=a.workload)
    prob = bench.Problem(w, 0, 1, 2)
    s = torch.cuda.Stream()
    ts = 128 * (32 if w["dtype"] == "f32" else 16) * (2 if w["order"] >= 4 else 1)   # tile samples (lti.cuh Chunk)
    ntot = w["batch"] * ((w["length"] + ts - 1) // ts)
    buf = torch.zeros(ntot * 16 + 8, dtype=torch.int64, device="cuda")
    buf2 = torch.zeros(ntot * 16 + 8, dtype=torch.int64, device="cuda")

    def reset(b):
        b.zero_()
        b[ntot * 16::2] = (1 << 63) - 1          # span entry slots (atomicMin)
    for rep in range(a.reps):
        with torch.cuda.stream(s):
            prob.step(0, s)
        torch.cuda.synchronize()
    # one whole step (prep, fwd, bwd back to back on one stream): kernel spans
    st = prob.sets[0]
    for rep in range(3):
        reset(buf)
        reset(buf2)
        with torch.cuda.stream(s):
            B.iir_debug_trace(buf)
            B.iir_forward(prob.desc, prob.b, prob.a, st["x"], prob.zi, st["y"], prob.zf, prob.tape, prob.tb,
                          prob.ws, prob.wb, s)
            B.iir_debug_trace(buf2)
            B.iir_backward(prob.desc, st["gy"], prob.gzf, prob.b, prob.a, st["x"], st["y"], prob.zi, prob.tape,
                           prob.tb, st["gx"], prob.gb, prob.ga, prob.gzi, prob.ws, prob.wb, s)
            B.iir_debug_trace(None)
        torch.cuda.synchronize()
    # the same step captured in a CUDA graph (the bench's timed mode: PDL overlaps the launches)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        B.iir_debug_trace(buf)
        B.iir_forward(prob.desc, prob.b, prob.a, st["x"], prob.zi, st["y"], prob.zf, prob.tape, prob.tb,
                      prob.ws, prob.wb, s)
        B.iir_debug_trace(buf2)
        B.iir_backward(prob.desc, st["gy"], prob.gzf, prob.b, prob.a, st["x"], st["y"], prob.zi, prob.tape,
                       prob.tb, st["gx"], prob.gb, prob.ga, prob.gzi, prob.ws, prob.wb, s)
        B.iir_debug_trace(None)
    torch.cuda.synchronize()
    for rep in range(3):
        reset(buf)
        reset(buf2)
        gr.replay()
        torch.cuda.synchronize()
    g1 = buf[ntot * 16:].cpu().numpy().astype(np.float64)
    g2 = buf2[ntot * 16:].cpu().numpy().astype(np.float64)
    gt0 = g1[0]
    print("== one step in a CUDA graph, kernel spans (us from prep entry): " + ", ".join(
        f"{k} [{(v[0] - gt0) / 1e3:.2f}, {(v[1] - gt0) / 1e3:.2f}]" for k, v in
        {"prep": (g1[0], g1[1]), "fwd": (g1[2], g1[3]), "bwd": (g2[4], g2[5])}.items()))
    reset(buf)
    reset(buf2)
    with torch.cuda.stream(s):
        B.iir_debug_trace(buf)
        B.iir_forward(prob.desc, prob.b, prob.a, st["x"], prob.zi, st["y"], prob.zf, prob.tape, prob.tb,
                      prob.ws, prob.wb, s)
        B.iir_debug_trace(buf2)
        B.iir_backward(prob.desc, st["gy"], prob.gzf, prob.b, prob.a, st["x"], st["y"], prob.zi, prob.tape,
                       prob.tb, st["gx"], prob.gb, prob.ga, prob.gzi, prob.ws, prob.wb, s)
        B.iir_debug_trace(None)
    torch.cuda.synchronize()
    a1 = buf[ntot * 16:].cpu().numpy().astype(np.float64)
    a2 = buf2[ntot * 16:].cpu().numpy().astype(np.float64)
    t0 = a1[0]
    spans = {"prep": (a1[0], a1[1]), "fwd": (a1[2], a1[3]), "bwd": (a2[4], a2[5])}
    print("== one step, kernel spans (us from prep entry): " + ", ".join(
        f"{k} [{(v[0] - t0) / 1e3:.2f}, {(v[1] - t0) / 1e3:.2f}]" for k, v in spans.items()))
    tf = buf[:ntot * 16].view(ntot, 16).cpu().numpy().astype(np.float64)
    tb_ = buf2[:ntot * 16].view(ntot, 16).cpu().numpy().astype(np.float64)
    for k, nm in ((8, "partial"), (9, "group"), (12, "set-start"), (13, "set-sum"), (14, "chain"), (10, "pre-exit"),
                  (11, "exit")):
        col = tb_[:, k]
        col = col[col > 0]
        if col.size:
            print(f"   bwd {nm:9s} max {(col.max() - t0) / 1e3:.2f}  n={col.size}")
    print("   fwd tiles: first start %.2f last store %.2f | bwd tiles: first start %.2f last store %.2f" % (
        (tf[:, 0].min() - t0) / 1e3, (tf[:, 5].max() - t0) / 1e3, (tb_[:, 0].min() - t0) / 1e3,
        (tb_[:, 5].max() - t0) / 1e3))
    for kern in ("fwd", "bwd"):
        reset(buf)
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
        t = buf[:ntot * 16].view(ntot, 16).cpu().numpy().astype(np.float64)
        t0 = t[:, 0].min()
        rel = (t - t0) / 1e3
        names = PH_F if kern == "fwd" else PH_B
        print(f"== {kern} ({ntot} tiles), us relative to first tile start; columns p0 p10 p50 p90 p100")
        for k, nm in enumerate(names):
            col = rel[:, k]
            col = col[t[:, k] > 0]
            if nm == "-" or col.size == 0:
                continue
            q = np.percentile(col, [0, 10, 50, 90, 100])
            print(f"   {nm:8s} " + " ".join(f"{v:8.2f}" for v in q))
        d = np.diff(rel, axis=1)
        print("   phase durations (median us): " + ", ".join(
            f"{names[k]}->{names[k + 1]} {np.median(d[:, k]):.2f}" for k in range(5)))
        ok = (t[:, 6] > 0) & (t[:, 2] > 0)
        if ok.any():
            w0 = (t[ok, 6] - t[ok, 2]) / 1e3
            print("   scan->lvl0 wait p50 %.2f p90 %.2f" % tuple(np.percentile(w0, [50, 90])))
        ok = (t[:, 7] > 0) & (t[:, 6] > 0)
        if ok.any():
            w1 = (t[ok, 7] - t[ok, 6]) / 1e3
            w2 = (t[ok, 3] - t[ok, 7]) / 1e3
            print("   lvl0->lvl1 p50 %.2f p90 %.2f ; lvl1->carry p50 %.2f p90 %.2f" % (
                tuple(np.percentile(w1, [50, 90])) + tuple(np.percentile(w2, [50, 90]))))


if __name__ == "__main__":
    main()
