"""One whole step (iir_forward + iir_backward) bracketed by cudaProfilerStart/Stop, for an
in-situ DRAM count of the step with ncu range replay:

    ncu --replay-mode range --profile-from-start off \\
        --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \\
        python tools/step_range.py --workload c5

The range replays the step's launches together (PDL overlap and L2 state between the
kernels as in a real step), unlike the per-kernel cold replays of the launch lists."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c5")
    a = ap.parse_args()
    w = dict(bench.WORKLOADS[a.workload], key=a.workload, engine="auto")
    prob = bench.Problem(w, 0, 1, 3)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3):
            prob.step(i, s)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    with torch.cuda.stream(s):
        prob.step(0, s)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    samples = w["batch"] * w["length"]
    print(f"{a.workload}: one step of {samples} samples inside the profiler range")


if __name__ == "__main__":
    main()
