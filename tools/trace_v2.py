"""Per-tile phase timeline of the round-2 LTI kernels (iir_debug_trace): where a tile's
time goes.   python tools/trace_v2.py [--workload c5]
Stamps per tile: [0] aggregate start [1] data ready [2] published [3] look-back start
[4] carry known [5] emit done [6] stored [7] warp."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2511_14390_b200 import _binding as B  # noqa: E402


def summarize(name, tr, ntot):
    t = tr[:ntot * 8].reshape(ntot, 8).astype(np.int64)
    c = tr[ntot * 8:].reshape(-1, 8).astype(np.int64)
    c = c[c[:, 0] > 0]
    t = t[t[:, 0] > 0]
    t0 = min(t[:, 0].min(), c[:, 0].min()) if len(c) else t[:, 0].min()
    if len(c):
        cs = (c[:, :4] - t0) / 1e3
        print(f"== {name}: {len(c)} CTAs: entry p50 {np.median(cs[:, 0]):.2f} max {cs[:, 0].max():.2f}; setup done p50 "
              f"{np.median(cs[:, 1]):.2f} max {cs[:, 1].max():.2f}; tiles done p50 {np.median(cs[:, 2]):.2f} max "
              f"{cs[:, 2].max():.2f}; exit p50 {np.median(cs[:, 3]):.2f} max {cs[:, 3].max():.2f} us")
        if (c[:, 4] > 0).any():
            c4 = (c[:, 4:6] - t0) / 1e3
            i = int(np.argmax(cs[:, 3]))
            print(f"   finalize done p50 {np.median(c4[:, 0]):.2f} max {c4[:, 0].max():.2f}; cta_exit done p50 "
                  f"{np.median(c4[:, 1]):.2f} max {c4[:, 1].max():.2f}; last CTA {i}: tiles {cs[i, 2]:.2f} "
                  f"finalize {c4[i, 0]:.2f} cta_exit {c4[i, 1]:.2f} exit {cs[i, 3]:.2f} us")
        ntot = len(t)
    st = (t[:, :7] - t0) / 1e3                     # us
    span = (t[:, 6].max() - t0) / 1e3
    d = {"data wait": st[:, 1] - st[:, 0], "aggregate": st[:, 2] - st[:, 1], "until look-back": st[:, 3] - st[:, 2],
         "look-back": st[:, 4] - st[:, 3], "emit": st[:, 5] - st[:, 4], "store/partials": st[:, 6] - st[:, 5],
         "tile life": st[:, 6] - st[:, 0]}
    print(f"== {name}: {ntot} tiles, span {span:.1f} us, warps {len(np.unique(t[:, 7]))}")
    for k, v in d.items():
        print(f"   {k:16s} p10 {np.percentile(v, 10):7.2f}  p50 {np.percentile(v, 50):7.2f}  p90 {np.percentile(v, 90):7.2f}"
              f"  mean {v.mean():7.2f} us")
    late = np.argsort(st[:, 6])[-8:]
    for i in late:
        print(f"   late tile (row {i}, warp {t[i, 7]}): start {st[i, 0]:.1f} data {st[i, 1]:.1f} pub {st[i, 2]:.1f} "
              f"lb {st[i, 3]:.1f} carry {st[i, 4]:.1f} emit {st[i, 5]:.1f} stored {st[i, 6]:.1f}")
    w = t[:, 7]
    per = np.bincount(w.astype(np.int64))
    print(f"   tiles per warp: min {per[per > 0].min()} max {per.max()}")
    first = np.sort(st[:, 0])
    print(f"   aggregate starts: first {first[0]:.1f}, 10% {np.percentile(first, 10):.1f}, 90% {np.percentile(first, 90):.1f}, last {first[-1]:.1f} us")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--engine", default="auto")
    a = ap.parse_args()
    w = dict(bench.WORKLOADS[a.workload], key=a.workload, engine=a.engine)
    prob = bench.Problem(w, 0, 1, 2)
    s = torch.cuda.Stream()
    ts = 32 * int(os.environ.get("IIRG_V2_L", "64"))
    ntot = w["batch"] * ((w["length"] + ts - 1) // ts)
    half = (ntot + 4096) * 8                      # tile stamps, then CTA stamps
    buf = torch.zeros(half, dtype=torch.int64, device="cuda")
    buf2 = torch.zeros(half, dtype=torch.int64, device="cuda")
    for rep in range(3):
        with torch.cuda.stream(s):
            prob.step(0, s)
    torch.cuda.synchronize()
    st = prob.sets[0]
    for rep in range(2):
        buf.zero_(); buf2.zero_()
        with torch.cuda.stream(s):
            B.iir_debug_trace(buf)
            B.iir_forward(prob.desc, prob.b, prob.a, st["x"], prob.zi, st["y"], prob.zf, prob.tape, prob.tb,
                          prob.ws, prob.wb, s)
            B.iir_debug_trace(buf2)
            B.iir_backward(prob.desc, st["gy"], prob.gzf, prob.b, prob.a, st["x"], st["y"], prob.zi, prob.tape,
                           prob.tb, st["gx"], prob.gb, prob.ga, prob.gzi, prob.ws, prob.wb, s)
            B.iir_debug_trace(None)
        torch.cuda.synchronize()
    summarize("forward", buf.cpu().numpy(), ntot)
    summarize("backward", buf2.cpu().numpy(), ntot)


if __name__ == "__main__":
    main()
