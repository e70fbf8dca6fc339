"""Benchmark of the hot path: forward + backward IIR filtering (BASELINE.json metric
"fwd+bwd filtered samples/sec (B x T / s) and HBM GB/s vs peak").

    python bench.py [--gpus N --steps K --warmup W] [--workload c5|c2|c1|c4|c3|f1|f2|f3]
                    [--scaling weak|strong] [--impl ours|reference]

Default workload: BASELINE.json's config 5 (order-8 TDF, shared coefficients,
2^16-sample sequences, coefficient-gradient all-reduce), the configuration the
metric's 1/2/4/8-GPU figure is quoted on: weak scaling (default) runs 256
sequences per GPU (2048 at G = 8); --scaling strong splits the global batch of
2048 over the G ranks.  `--gpus N` with N > 1 launched without torchrun
re-launches itself under `torch.distributed.run` (N ranks, one per GPU, NCCL).

One step = iir_forward + iir_backward (all of SURVEY §8(a)'s rows a1-a8) over one
batch of synthetic input already resident in HBM, plus (N > 1) the NCCL
all-reduce of the shared-coefficient gradients (dist.reduce_shared_grads, the
product's driver).  Inputs rotate over several buffer sets
whose total size exceeds 2x L2, so no step reads data left in L2 by the
previous one.  The timed region is K steps captured in one CUDA graph (eager
with --no-graph), bracketed by barrier + synchronize, timed with CUDA events on
the launching stream, max over ranks.  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2511_14390_b200 import inputs  # noqa: E402

METRIC = "fwd+bwd filtered samples/sec (B x T / s)"
WORKLOADS = {
    "c1": dict(desc="config 1: order-2 TDF biquad, batch 1 x 4096, fixed coefficients, fp64", **inputs.CONFIGS["c1"]),
    "c2": dict(desc="config 2: order-2 TDF fixed coefficients, batch 64 x 2^16, fp32 (audio EQ training shape)",
               **inputs.CONFIGS["c2"]),
    "c4": dict(desc="config 4: order-4 TDF, batch 1 x 2^24, fp32 (time-parallel scan stress)", **inputs.CONFIGS["c4"]),
    "c5": dict(desc="config 5 per-GPU shard: order-8 TDF shared coefficients, batch 256 x 2^16 per GPU, fp32, "
                    "coefficient-gradient all-reduce", **dict(inputs.CONFIGS["c5"], batch=256)),
    "c3": dict(desc="config 3: all-pole LPC order 24, per-sample coefficients, batch 32 x 2^18, fp32",
               **inputs.CONFIGS["c3"]),
    "f2": dict(desc="SURVEY 8(f) f2: general time-varying DF (per-sample b and a), config-3 shape: order 24, "
                    "batch 32 x 2^18, fp32", fir=True, **inputs.CONFIGS["c3"]),
    "f2t": dict(desc="SURVEY 8(f) f2: general time-varying TDF-II (per-sample b and a, DESIGN.md R20), config-3 "
                     "shape: order 24, batch 32 x 2^18, fp32", fir=True, **dict(inputs.CONFIGS["c3"], form="tdf")),
    "f1": dict(desc="SURVEY 8(f) f1: bare recurrence v(n+1) = A v(n) + z(n) of Listing 1, M = 2, batch 16 x 2^20, "
                    "fp32 (the paper's benchmarked operator at its longest N)", **dict(inputs.CONFIGS["f1"], batch=16)),
    "f3": dict(desc="SURVEY 8(f) f3: Diag-EXT bare recurrence (eigen-basis element-wise complex scans), f1's shape: "
                    "M = 2, batch 16 x 2^20, fp32", diag=True, **dict(inputs.CONFIGS["f1"], batch=16)),
    # PAPER.md:167 "we expect the gap [Diag-EXT vs EXT] to disappear as M increases": the same pair at M = 4
    # the DF-II form of config 5 (round-1 engine; u re-run in the backward from the tape's chunk states)
    "c5df": dict(desc="config 5 per-GPU shard in DF-II form: order-8 DF shared coefficients, batch 256 x 2^16, fp32",
                 **dict(inputs.CONFIGS["c5"], batch=256, form="df")),
    "f1m4": dict(desc="SURVEY 8(f) f1 at M = 4: dense bare recurrence, batch 16 x 2^20, fp32",
                 **dict(inputs.CONFIGS["f1"], batch=16, order=4)),
    "f3m4": dict(desc="SURVEY 8(f) f3 at M = 4: Diag-EXT bare recurrence, batch 16 x 2^20, fp32", diag=True,
                 **dict(inputs.CONFIGS["f1"], batch=16, order=4)),
}


def algorithmic_bytes(w):
    """Bytes per sample the method must move, per kernel."""
    s = 8 if w["dtype"] == "f64" else 4
    if w["form"] == "ss" and w.get("diag"):
        # diag_agg reads z (fwd) / gv (bwd); diag_fwd reads z, writes v; diag_bwd reads gv, v, writes gz;
        # diag_prep / diag_scan / diag_red touch per-set and per-chunk data only
        M = w["order"]
        return {"diag_prep": 0, "diag_agg": M * s, "diag_scan": 0, "diag_fwd": 2 * M * s, "diag_bwd": 3 * M * s,
                "diag_red": 0}
    if w["form"] == "ss":                       # rec_fwd reads z, writes v; rec_bwd reads gv, v, writes gz
        return {"rec_fwd": 2 * w["order"] * s, "rec_bwd": 3 * w["order"] * s}
    if w["coef"] == "per_sample":
        # tv_phi reads a, x; tv_fwd reads a, x and writes y; tv_bwd_agg reads a, dy;
        # tv_bwd reads a, dy, y and writes dx, grad_a.  tv_chain moves only the
        # per-segment tape (M^2 per 512 samples): design overhead, no per-sample bytes.
        M = w["order"]
        # tv_wagg: the fp64 re-run of the segments' zero-state responses (reads a, x; beside tv_phi)
        d = {"tv_phi": (M + 1) * s, "tv_wagg": (M + 1) * s, "tv_chain": 0, "tv_fwd": (M + 2) * s,
             "tv_bwd_agg": (M + 1) * s, "tv_bwd": (2 * M + 3) * s}
        if w.get("fir"):       # FIR stage, 3 launches per step: fwd b, u -> y; bwd b, dy, u -> du, grad_b; zi add
            d["tv_fir"] = ((M + 3) + (2 * M + 5)) * s / 3
        if w.get("fir") and w["form"] == "tdf":   # TDF: skew of a / unskew of grad_a~ (design overhead;
            d["tv_skew"] = 4 * M * s             # b is read at skewed rows in place): read + write each
        return d
    # HBM bytes per kernel the method must move: fwd reads x, writes y; bwd reads dy, x, y (TDF:
    # 24 B/sample in fp32) or dy, x (DF: u re-run from the tape's chunk states, 20 B/sample) and writes dx
    if w["form"] == "tdf":
        return dict(lti_fwd=2 * s, lti_bwd=4 * s)
    return dict(lti_fwd=2 * s, lti_bwd=3 * s)


def step_min_bytes(w):
    """HBM bytes per sample any fwd+bwd implementation must move:
    LTI TDF x, y, dy, dx (+x, y re-read by the backward; DF +x only); TV all-pole x, y, dy, dx,
    a read by each direction and grad_a written: (3M + 5) elements."""
    s = 8 if w["dtype"] == "f64" else 4
    if w["form"] == "ss":
        return 5 * w["order"] * s
    if w["coef"] == "per_sample":
        # + per-sample b read by each direction and grad_b written (general DF)
        return (3 * w["order"] + 5 + (3 * (w["order"] + 1) if w.get("fir") else 0)) * s
    return (6 if w["form"] == "tdf" else 5) * s     # DF: x, y, dy, x, dx (u is not stored)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


class ClockSampler:
    """Samples SM clock + throttle reasons with NVML every ~2 ms in a thread."""

    def __init__(self, dev_index):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)

    _NAMES = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
              0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._NAMES.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.0005)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------ ours ---
class Problem:
    """Device-resident buffers of one workload for the C-ABI calls."""

    def __init__(self, w, dev, seed, nsets):
        from paper_2511_14390_b200 import _binding as B
        self.B = B
        self.w = w
        td = inputs.torch_dtype(w["dtype"])
        Bsz, T, M = w["batch"], w["length"], w["order"]
        rng = np.random.default_rng(1000)          # coefficients: the same on every rank (SHARED filter)
        self.td = td
        g = torch.Generator(device=dev).manual_seed(seed)
        self.sets = []
        ss = w["form"] == "ss"
        shape = (Bsz, T, M) if ss else (Bsz, T)
        if w["coef"] == "per_sample":
            if w.get("fir"):
                p = inputs.tv_df_problem(seed, batch=Bsz, length=T, order=M, dtype=w["dtype"], device=dev)
            else:
                p = inputs.tv_allpole_problem(seed, batch=Bsz, length=T, order=M, dtype=w["dtype"], device=dev)
            self.a = p["a"].to(td).contiguous()
            self.b = p["b"].to(td).contiguous() if w.get("fir") else None
            self.zi = p["zi"].to(td).contiguous()
            mode = B.IIR_COEF_PER_SAMPLE
        elif ss:
            self.a = torch.tensor(inputs.stable_matrix(rng, M), dtype=td, device=dev)
            self.b = None
            self.zi = (0.1 * torch.randn(Bsz, M, generator=g, device=dev, dtype=torch.float64)).to(td)
            mode = B.IIR_COEF_SHARED
        else:
            b, a = inputs.stable_coefs(rng, M, w["dtype"], angles=w["angles"])
            self.b = torch.tensor(b, dtype=td, device=dev)
            self.a = torch.tensor(a, dtype=td, device=dev)
            self.zi = (0.1 * torch.randn(Bsz, M, generator=g, device=dev, dtype=torch.float64)).to(td)
            mode = B.IIR_COEF_SHARED
        self.gzf = None if ss else torch.randn(Bsz, M, generator=g, device=dev, dtype=torch.float64).to(td)
        for _ in range(nsets):
            x = torch.randn(*shape, generator=g, device=dev, dtype=td)
            gy = torch.randn(*shape, generator=g, device=dev, dtype=td)
            st = dict(x=x, gy=gy, y=torch.empty_like(x), gx=torch.empty_like(x))
            if w["coef"] == "per_sample":
                st["ga"] = torch.empty_like(self.a)          # (B, T, M): one per set, like y and dx
            self.sets.append(st)
        self.zf = None if ss else torch.empty(Bsz, M, dtype=td, device=dev)
        self.gzi = torch.empty(Bsz, M, dtype=td, device=dev)
        self.gb = None if self.b is None else torch.empty_like(self.b)
        self.ga = None if w["coef"] == "per_sample" else torch.empty_like(self.a)
        # the workspace is cleared once; every completed call leaves it cleared
        # engine: auto (by order), v1 (round-1 CTA tiles), v2 (round-2 persistent warp tiles);
        # grad_y is resident before the step: the backward may read it while the forward drains
        sched = {"auto": 0, "v1": B.IIR_FLAG_LEGACY_LTI, "v2": B.IIR_FLAG_ENGINE_V2}[w.get("engine", "auto")]
        sched |= B.IIR_FLAG_GRAD_Y_EARLY
        if w.get("fir"):
            sched |= B.IIR_FLAG_PER_SAMPLE_B
        if w.get("diag"):
            sched |= B.IIR_FLAG_DIAG
        self.desc = B.make_desc(Bsz, T, M, w["form"], td, mode, flags=B.IIR_FLAG_WS_READY | sched)
        self.tb = B.iir_tape_bytes(self.desc)
        self.wb = B.iir_workspace_bytes(self.desc)
        self.tape = torch.empty(self.tb, dtype=torch.uint8, device=dev)
        self.ws = torch.empty(self.wb, dtype=torch.uint8, device=dev)
        B.iir_workspace_init(self.desc, self.ws, self.wb, torch.cuda.current_stream(dev))
        self.grad_buf = None if self.b is None else torch.empty(2 * (M + 1), dtype=td, device=dev)
        self.ss = ss

    def set_bytes(self):
        s = self.sets[0]
        return sum(t.numel() * t.element_size() for t in s.values())

    def step(self, i, stream, pg=None):
        B = self.B
        s = self.sets[i % len(self.sets)]
        B.iir_forward(self.desc, self.b, self.a, s["x"], self.zi, s["y"], self.zf, self.tape, self.tb,
                      self.ws, self.wb, stream)
        B.iir_backward(self.desc, s["gy"], self.gzf, self.b, self.a, s["x"], s["y"], self.zi, self.tape, self.tb,
                       s["gx"], self.gb, s.get("ga", self.ga), self.gzi, self.ws, self.wb, stream)
        if pg is not None and self.b is not None and self.w["coef"] == "shared":
            # the one real exchange of the path: all-reduce of the shared-coefficient gradients (§8(e)),
            # through the product's batch-sharded driver
            from paper_2511_14390_b200 import dist as D
            D.reduce_shared_grads(self.gb, self.ga, group=pg)
        elif pg is not None and self.ss:
            torch.distributed.all_reduce(self.ga, group=pg)      # shared A of the bare recurrence


def run_ours(args, w, rank, world, dev, pg):
    from paper_2511_14390_b200 import _binding as B
    torch.cuda.set_device(dev)
    L2 = torch.cuda.get_device_properties(dev).L2_cache_size
    samples = w["batch"] * w["length"]
    bytes_per_set = 4 * samples * (8 if w["dtype"] == "f64" else 4) * (w["order"] if w["form"] == "ss" else 1)
    nsets = max(2, int(np.ceil(3 * L2 / bytes_per_set)) + 1)
    nsets = min(nsets, 64)
    prob = Problem(w, dev, 1000 + rank, nsets)
    stream = torch.cuda.Stream(device=dev)
    use_graph = not args.no_graph

    def run_steps(i0, n):
        for i in range(i0, i0 + n):
            prob.step(i, stream, pg)

    with torch.cuda.stream(stream):
        run_steps(0, max(args.warmup, 1))           # warm-up (also sets kernel attributes)
    torch.cuda.synchronize(dev)

    graph = None
    if use_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                run_steps(args.warmup, args.steps)
            torch.cuda.synchronize(dev)
            stream.wait_stream(torch.cuda.current_stream(dev))
            for _ in range(max(args.warmup, 3)):   # warm replays
                with torch.cuda.stream(stream):
                    graph.replay()
            torch.cuda.synchronize(dev)
        except Exception as e:  # pragma: no cover - fall back to eager on capture failure
            print(f"[bench] graph capture failed ({e}); timing eager launches", file=sys.stderr)
            graph = None
            use_graph = False

    # ---- timed region ----
    sampler = ClockSampler(dev if isinstance(dev, int) else torch.cuda.current_device())
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    launches0 = B.iir_launch_count()
    with sampler:
        with torch.cuda.stream(stream):
            e0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                run_steps(args.warmup, args.steps)
            e1.record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    ms = e0.elapsed_time(e1)
    # kernels per step are counted at capture/eager time
    per_step_launches = None
    if graph is None:
        gpu_launches = B.iir_launch_count() - launches0
    else:
        n0 = B.iir_launch_count()
        with torch.cuda.stream(stream):
            prob.step(0, stream, None)
        torch.cuda.synchronize(dev)
        per_step_launches = B.iir_launch_count() - n0
        gpu_launches = per_step_launches * args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    ms = float(t.item())

    # ---- per-kernel device times: the same K steps, each launch bracketed by
    #      CUDA events on its stream (library instrumentation), eager ----
    # Per-kernel device times: every library launch bracketed by CUDA events on
    # its stream.  The K steps are captured in a CUDA graph with the events (as
    # in the timed region, no host submission gaps inside an event pair; the
    # event nodes do serialise the launches, so PDL overlap is not counted) and
    # replayed once.  Eager launching (--no-graph) records them directly.
    B.iir_profile_reset()
    B.iir_profile_enable(True)
    if use_graph and world == 1:        # multi-rank runs profile eagerly (no second NCCL capture)
        pg_graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(pg_graph, stream=stream):
            run_steps(args.warmup, args.steps)
        torch.cuda.synchronize(dev)
        with torch.cuda.stream(stream):
            pg_graph.replay()
    else:
        with torch.cuda.stream(stream):
            run_steps(args.warmup, args.steps)
    torch.cuda.synchronize(dev)
    B.iir_profile_enable(False)
    names = B.kernel_names()
    ktimes = {}
    for k, nm in enumerate(names):
        tot, n = B.iir_profile_query(k)
        if n:
            ktimes[nm] = (tot, n)
    B.iir_profile_reset()

    # ---- e2e: through the public API with HOST buffers (pinned), copies inside the timed region ----
    e2e = run_e2e(args, prob, stream, dev, world)

    return dict(ms=ms, ktimes=ktimes, gpu_launches=gpu_launches, per_step_launches=per_step_launches,
                clocks=sampler.summary(), nsets=nsets, set_bytes=prob.set_bytes(), L2=L2, graph=use_graph,
                e2e=e2e)


def run_e2e(args, prob, stream, dev, world):
    """Every step: H2D of x, dy from pinned host memory, fwd + bwd through the C
    ABI, D2H of y, dx and the small outputs.  Three streams pipeline the steps
    (H2D of step i+1 and D2H of step i-1 overlap the kernels of step i) over two
    device buffer sets; every copy of every step is inside the timed region."""
    nbuf = min(2, len(prob.sets))
    hx = [torch.empty_like(prob.sets[0]["x"], device="cpu").pin_memory() for _ in range(nbuf)]
    hgy = [torch.empty_like(prob.sets[0]["gy"], device="cpu").pin_memory() for _ in range(nbuf)]
    for i in range(nbuf):
        hx[i].copy_(prob.sets[i]["x"])
        hgy[i].copy_(prob.sets[i]["gy"])
    big = ["y", "gx"] + (["ga"] if "ga" in prob.sets[0] else [])
    hbig = [{k: torch.empty_like(prob.sets[0][k], device="cpu").pin_memory() for k in big} for _ in range(nbuf)]
    outs_small = [t for t in (prob.gb, prob.ga, prob.zf, prob.gzi) if t is not None]
    hsmall = [[torch.empty_like(t, device="cpu").pin_memory() for t in outs_small] for _ in range(nbuf)]
    small_dev = [[torch.empty_like(t) for t in outs_small] for _ in range(nbuf)]
    steps = max(3, min(args.steps, 20))
    s_h2d = torch.cuda.Stream(device=dev)
    s_d2h = torch.cuda.Stream(device=dev)
    s_h2d2 = torch.cuda.Stream(device=dev)       # second copy of each direction runs concurrently
    s_d2h2 = torch.cuda.Stream(device=dev)
    ev = lambda: torch.cuda.Event()
    h2d_done = [ev() for _ in range(nbuf)]
    comp_done = [ev() for _ in range(nbuf)]
    d2h_done = [ev() for _ in range(nbuf)]
    used = [False] * nbuf

    def one(i):
        k = i % nbuf
        s = prob.sets[k]
        with torch.cuda.stream(s_h2d):
            if used[k]:
                s_h2d.wait_event(comp_done[k])          # the kernels of step i-2 have read set k
            s_h2d2.wait_stream(s_h2d)
            s["x"].copy_(hx[k], non_blocking=True)
            with torch.cuda.stream(s_h2d2):
                s["gy"].copy_(hgy[k], non_blocking=True)
            s_h2d.wait_stream(s_h2d2)
            h2d_done[k].record(s_h2d)
        stream.wait_event(h2d_done[k])
        if used[k]:
            stream.wait_event(d2h_done[k])              # y, dx of step i-2 have left the device
        with torch.cuda.stream(stream):
            prob.step(k, stream, None)
            for d, t in zip(small_dev[k], outs_small):
                d.copy_(t, non_blocking=True)
            comp_done[k].record(stream)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(comp_done[k])
            s_d2h2.wait_stream(s_d2h)
            for j, name in enumerate(big):
                with torch.cuda.stream(s_d2h2 if j % 2 else s_d2h):
                    hbig[k][name].copy_(s[name], non_blocking=True)
            for h, d in zip(hsmall[k], small_dev[k]):
                h.copy_(d, non_blocking=True)
            s_d2h.wait_stream(s_d2h2)
            d2h_done[k].record(s_d2h)
        used[k] = True

    one(0)
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s_h2d)
    stream.wait_stream(s_h2d)
    s_d2h.wait_stream(s_h2d)
    for i in range(1, steps + 1):
        one(i)
    s_h2d.wait_stream(s_d2h)
    s_h2d.wait_stream(stream)
    e1.record(s_h2d)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / steps
    h2d = hx[0].numel() * hx[0].element_size() + hgy[0].numel() * hgy[0].element_size()
    d2h = sum(h.numel() * h.element_size() for h in list(hbig[0].values()) + hsmall[0])
    return dict(ms_per_step=ms, h2d=h2d, d2h=d2h, steps=steps, pipelined=True)


def cpu_baseline(w, budget_s=10.0):
    """The fp64 oracle as it stands, on the host cores, on a bounded sample."""
    import oracle
    oracle.build()
    rng = np.random.default_rng(7)
    T = w["length"]
    nseq = min(w["batch"], 64)
    what = "fp64 C oracle (dense state space)"
    if w["form"] == "ss" and w.get("diag"):
        from oracle import diag as odiag
        T = min(T, 1 << 16)
        nseq = 1
        p = inputs.rec_problem(7, batch=nseq, length=T, order=w["order"], dtype=w["dtype"])
        fn = lambda: odiag.diag_recurrence(p["A"], p["v0"][0], p["z"][0], p["gv"][0])
        what = "numpy complex128 Diag-EXT oracle (oracle/diag.py)"
    elif w["form"] == "ss":
        T = min(T, 1 << 20)
        nseq = 2
        p = inputs.rec_problem(7, batch=nseq, length=T, order=w["order"], dtype=w["dtype"])
        fn = lambda: [oracle.recurrence(p["A"], p["v0"][i], p["z"][i], p["gv"][i]) for i in range(nseq)]
    elif w["coef"] == "per_sample":
        T = min(T, 1 << 16)
        if w.get("fir"):
            p = inputs.tv_df_problem(7, batch=min(nseq, 8), length=T, order=w["order"], dtype=w["dtype"])
            args = tuple(p[k].numpy() for k in ("b", "a", "x", "zi", "gy", "gzf"))
            fn = lambda: oracle.tv_df(*args)
        else:
            p = inputs.tv_allpole_problem(7, batch=min(nseq, 8), length=T, order=w["order"], dtype=w["dtype"])
            args = (p["a"].numpy(), p["x"].numpy(), p["zi"].numpy(), p["gy"].numpy(), p["gzf"].numpy())
            fn = lambda: oracle.tv_allpole(*args)
        nseq = p["x"].shape[0]
    else:
        T = min(T, 1 << 20)
        nseq = max(1, min(nseq, (1 << 22) // T))
        p = inputs.lti_problem(7, form=w["form"], order=w["order"], batch=nseq, length=T, dtype=w["dtype"],
                               angles=w["angles"])
        form = 1 if w["form"] == "tdf" else 0
        fn = lambda: oracle.lti(form, p["b"], p["a"], p["x"], p["zi"], p["gy"], p["gzf"])
    cores = 1 if w["form"] == "ss" else min(os.cpu_count() or 1, nseq)
    reps = 0
    t0 = time.perf_counter()
    while True:
        fn()
        reps += 1
        el = time.perf_counter() - t0
        if el >= budget_s or (reps >= 1 and el * (reps + 1) / reps > 3 * budget_s):
            break
    value = reps * nseq * T / el
    return dict(value=value, unit="samples/s", cores=cores, kind="oracle",
                sample=f"{reps} x ({nseq} sequences x {T} samples) of the workload, {what}, "
                       f"{cores} host threads, {el:.1f} s wall")


# -------------------------------------------------------------- reference ---
def run_reference(args, w, rank, world):
    """--impl reference: the oracle (the reference arm of this tier) timed as
    the main loop, each step a bounded sample of the workload."""
    import oracle
    oracle.build()
    if rank != 0:
        return
    T = w["length"]
    if w["form"] == "ss" and w.get("diag"):
        from oracle import diag as odiag
        T = min(T, 1 << 15)
        nseq = 1
        p = inputs.rec_problem(7, batch=nseq, length=T, order=w["order"], dtype=w["dtype"])
        fn = lambda: odiag.diag_recurrence(p["A"], p["v0"][0], p["z"][0], p["gv"][0])
    elif w["form"] == "ss":
        T = min(T, 1 << 19)
        nseq = 1
        p = inputs.rec_problem(7, batch=nseq, length=T, order=w["order"], dtype=w["dtype"])
        fn = lambda: oracle.recurrence(p["A"], p["v0"][0], p["z"][0], p["gv"][0])
    elif w["coef"] == "per_sample":
        T = min(T, 1 << 15)
        nseq = min(w["batch"], 8)
        if w.get("fir"):
            p = inputs.tv_df_problem(7, batch=nseq, length=T, order=w["order"], dtype=w["dtype"])
            a_ = tuple(p[k].numpy() for k in ("b", "a", "x", "zi", "gy", "gzf"))
            fn = lambda: oracle.tv_df(*a_)
        else:
            p = inputs.tv_allpole_problem(7, batch=nseq, length=T, order=w["order"], dtype=w["dtype"])
            a_ = (p["a"].numpy(), p["x"].numpy(), p["zi"].numpy(), p["gy"].numpy(), p["gzf"].numpy())
            fn = lambda: oracle.tv_allpole(*a_)
    else:
        T = min(T, 1 << 20)
        nseq = max(1, min(w["batch"], 8, (1 << 21) // T))
        p = inputs.lti_problem(7, form=w["form"], order=w["order"], batch=nseq, length=T, dtype=w["dtype"],
                               angles=w["angles"])
        form = 1 if w["form"] == "tdf" else 0
        fn = lambda: oracle.lti(form, p["b"], p["a"], p["x"], p["zi"], p["gy"], p["gzf"])
    for _ in range(args.warmup):
        fn()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        fn()
    el = time.perf_counter() - t0
    cores = 1 if w["form"] == "ss" else min(os.cpu_count() or 1, nseq)
    value = args.steps * nseq * T / el
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": w["desc"], "batch": w["batch"], "length": w["length"], "order": w["order"],
                       "form": w["form"], "coef": w["coef"]},
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": cores, "kind": "oracle",
                             "sample": f"each step: {nseq} sequences x {T} samples of the workload, fp64 C oracle"},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def load_traffic(w):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return {}
    try:
        d = json.load(open(p))
        return d.get(w["key"], {})
    except Exception:
        return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOADS))
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                    help="c5: weak = 256 sequences per GPU; strong = the global batch of 2048 split over the GPUs")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--engine", default="auto", choices=["auto", "v1", "v2"],
                    help="fp32 TDF engine: auto (by order), v1 (round-1 CTA tiles), v2 (round-2 warp tiles)")
    args = ap.parse_args()
    w = dict(WORKLOADS[args.workload], key=args.workload, engine=args.engine)

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run (the driver's own launch line)
        if args.impl == "ours" and torch.cuda.device_count() < args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} CUDA device(s) visible")
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "ours" and world != args.gpus:
        print(f"[bench] note: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)
    if args.workload == "c5":
        glob = inputs.CONFIGS["c5"]["batch"]
        w["batch"] = 256 if args.scaling == "weak" else max(1, glob // world)
        w["desc"] = (f"config 5: order-8 TDF shared coefficients, 2^16-sample sequences, fp32, "
                     f"coefficient-gradient all-reduce; {w['batch']} sequences per GPU x {world} GPU(s) "
                     f"({args.scaling} scaling; global batch {w['batch'] * world})")

    if args.impl == "reference":
        run_reference(args, w, rank, world)
        return

    pg = None
    if world > 1:
        torch.cuda.set_device(local)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = torch.distributed.group.WORLD
    dev = local
    r = run_ours(args, w, rank, world, dev, pg)

    samples_step = w["batch"] * w["length"] * world
    value = samples_step * args.steps / (r["ms"] * 1e-3)
    peak, peak_src = peaks()
    abytes = algorithmic_bytes(w)
    roof = None
    if r["ktimes"]:
        dom = max(r["ktimes"], key=lambda k: r["ktimes"][k][0])
        tot, n = r["ktimes"][dom]
        avg_ms = tot / n
        # a kind launched k times per step (three-phase mode) moves its bytes over k launches
        per_launch = abytes.get(dom, 0) * w["batch"] * w["length"] / max(1.0, n / args.steps)
        achieved = per_launch / (avg_ms * 1e-3) / 1e9
        tr = load_traffic(w).get(dom)
        step_kernel_ms = sum(t for t, _ in r["ktimes"].values()) / args.steps
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": tr, "peak_source": peak_src,
                "algorithmic_bytes_per_launch": per_launch, "avg_launch_ms": avg_ms,
                "launch_timing": "CUDA events around every library launch on its stream, the K steps captured "
                                 "with the events in a CUDA graph and replayed (event nodes serialise the "
                                 "launches: no PDL overlap counted)" if (r["graph"] and world == 1)
                                else "CUDA events, eager launches",
                "kernel_ms": {k: t / n_ for k, (t, n_) in r["ktimes"].items()},
                "share_of_step": {k: (t / args.steps) / step_kernel_ms for k, (t, _) in r["ktimes"].items()}}
    step_bytes = step_min_bytes(w) * w["batch"] * w["length"]
    e2e = r["e2e"]
    e2e_val = samples_step / (e2e["ms_per_step"] * 1e-3) if e2e else None
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w)
    line = {
        "metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["ms"] / args.steps, "higher_is_better": True,
        "scaling": args.scaling,
        "vs_baseline": None, "dtype": w["dtype"], "data": "synthetic (seeded Gaussian signals, random stable filters)",
        "config": {"workload": w["desc"], "batch_per_gpu": w["batch"], "global_batch": w["batch"] * world,
                   "length": w["length"], "order": w["order"],
                   "form": w["form"], "coef": w["coef"], "engine": w["engine"],
                   "l2": f"{r['nsets']} rotating input/output buffer sets x {r['set_bytes'] / 2**20:.0f} MiB "
                         f"(> 2x L2 = {2 * r['L2'] / 2**20:.0f} MiB)",
                   "timing": "CUDA graph of K steps" if r["graph"] else "eager launches",
                   "parallelism": f"dp{world} (batch-sharded)"},
        "hbm_gbs_algorithmic_step": step_bytes / (r["ms"] / args.steps * 1e-3) / 1e9,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "samples/s", "h2d_bytes_per_step": e2e["h2d"],
                "d2h_bytes_per_step": e2e["d2h"], "steps": e2e["steps"],
                "how": "pinned host buffers; H2D of x, dy and D2H of y, dx, zf, grad_zi, grad_b / grad_a every "
                       "step (per-sample a stays resident like weights), copies on two copy streams "
                       "overlapping the neighbouring steps' kernels"}
        if e2e else None,
        "gpu_launches": r["gpu_launches"],
        "clocks": r["clocks"],
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
