"""RBJ peaking-EQ stress set (reported, not gated).

The C2 shape (64 sequences x 2^16 samples, TDF-II order 2, fp32) with one RBJ cookbook
peaking EQ per sequence (PER_SEQ coefficients): f0 ~ log-U[20, 20000] Hz at 48 kHz,
Q ~ log-U[0.5, 8], gain ~ U[-12, 12] dB.  Low-frequency, high-Q sections put poles within
1e-3 of the unit circle, where fp32 arithmetic itself loses digits (the TDF
numerical-robustness remark this set probes).  For every sequence the GPU error of y and of
the gradients (normalised max error against the fp64 oracle, R13) is reported
next to the error of a plain fp32 sequential filter (scipy.signal.lfilter in float32) on
the same fp32-rounded inputs.

    python tools/rbj_stress.py [--out profiles/r02_rbj_stress.txt] [--batch 64] [--length 65536]
"""
import argparse
import os
import sys

import numpy as np
import scipy.signal as ss
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle  # noqa: E402
from paper_2511_14390_b200 import inputs  # noqa: E402
from gpu_util import nrm_err, run_lti_gpu  # noqa: E402


def problem(seed, batch, length):
    rng = np.random.default_rng(seed)
    f0 = np.exp(rng.uniform(np.log(20.0), np.log(20000.0), batch))
    q = np.exp(rng.uniform(np.log(0.5), np.log(8.0), batch))
    gain = rng.uniform(-12.0, 12.0, batch)
    bs, as_ = zip(*[inputs.rbj_peaking(f, qq, g) for f, qq, g in zip(f0, q, gain)])
    r32 = lambda v: np.asarray(v, np.float32).astype(np.float64)
    b, a = r32(np.stack(bs)), r32(np.stack(as_))
    x = r32(rng.standard_normal((batch, length)))
    gy = r32(rng.standard_normal((batch, length)))
    p = dict(form="tdf", b=b, a=a, x=x, gy=gy, zi=None, gzf=None, dtype="f32")
    return p, f0, q, gain


def run(batch=64, length=1 << 16, seed=4242):
    p, f0, q, gain = problem(seed, batch, length)
    g = run_lti_gpu(p)
    o = oracle.lti(1, p["b"], p["a"], p["x"], None, p["gy"], None)
    rows = []
    for i in range(batch):
        y32 = ss.lfilter(p["b"][i].astype(np.float32), p["a"][i].astype(np.float32), p["x"][i].astype(np.float32))
        # pole radius of the section
        r = float(np.max(np.abs(np.roots(p["a"][i]))))
        rows.append(dict(f0=f0[i], q=q[i], gain=gain[i], r=r,
                         gpu_y=nrm_err(g["y"][i], o["y"][i]), seq32_y=nrm_err(y32, o["y"][i]),
                         gpu_gx=nrm_err(g["gx"][i], o["gx"][i]),
                         gpu_gb=nrm_err(g["gb"][i], o["gb"][i]), gpu_ga=nrm_err(g["ga"][i], o["ga"][i])))
    return rows


def report(rows):
    lines = ["RBJ peaking-EQ stress set (SURVEY 8(d) C2 row; reported, not gated): 64 x 2^16 TDF-II biquads,",
             "one RBJ peaking EQ per sequence (PER_SEQ), fp32 GPU vs the fp64 oracle, next to fp32 sequential",
             "(scipy.signal.lfilter in float32) on the same inputs.  err = max|got - oracle| / rms(oracle).",
             "",
             f"{'f0 Hz':>9} {'Q':>5} {'gain dB':>7} {'1-r':>9} | {'gpu y':>9} {'fp32seq y':>9} | {'gpu gx':>9} {'gpu gb':>9} {'gpu ga':>9}"]
    for d in sorted(rows, key=lambda d: d["f0"]):
        lines.append(f"{d['f0']:9.1f} {d['q']:5.2f} {d['gain']:7.2f} {1 - d['r']:9.2e} | {d['gpu_y']:9.2e} "
                     f"{d['seq32_y']:9.2e} | {d['gpu_gx']:9.2e} {d['gpu_gb']:9.2e} {d['gpu_ga']:9.2e}")
    gy = np.array([d["gpu_y"] for d in rows])
    sy = np.array([d["seq32_y"] for d in rows])
    lines += ["",
              f"y error, GPU:            median {np.median(gy):.2e}  max {gy.max():.2e}",
              f"y error, fp32 sequential: median {np.median(sy):.2e}  max {sy.max():.2e}",
              f"sequences where the GPU error exceeds fp32 sequential: {int(np.sum(gy > sy))} of {len(rows)}",
              f"sequences above the 1e-4 gate: GPU {int(np.sum(gy > 1e-4))}, fp32 sequential {int(np.sum(sy > 1e-4))}"]
    return "\n".join(lines)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--length", type=int, default=1 << 16)
    a = ap.parse_args()
    assert torch.cuda.is_available(), "needs the GPU"
    txt = report(run(a.batch, a.length))
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt + "\n")


if __name__ == "__main__":
    main()
