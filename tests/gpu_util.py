"""Helpers of the GPU parity tests: run the CUDA path through the C ABI on a
generated problem, run the oracle on the same (dtype-rounded) inputs, and
compare tensor by tensor with the north-star error measure
max|gpu - oracle| / rms(oracle) (reading R13)."""
import numpy as np
import torch

import oracle
from paper_2511_14390_b200 import _binding as B

TOL = {"f32": 1e-4, "f64": 1e-10}


def nrm_err(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    if ref.size == 0:
        return 0.0
    s = float(np.sqrt(np.mean(ref ** 2)))
    return float(np.max(np.abs(got - ref))) / (s if s > 0 else 1.0)


def to_dev(a, dtype):
    if a is None:
        return None
    return torch.as_tensor(np.ascontiguousarray(a), dtype=torch.float64).to(dtype).cuda()


def run_lti_gpu(p, coef_mode=None, want=("y", "zf", "gx", "gb", "ga", "gzi"), repeat=1, stream=None, flags=0,
                flags_bwd=None):
    """Forward + backward through iir_forward / iir_backward.  Returns numpy fp64.
    `flags` (iir_flags_t, e.g. the scan schedule) for the forward; the backward
    uses `flags_bwd` when given, else the same."""
    td = torch.float32 if p["dtype"] == "f32" else torch.float64
    x = to_dev(p["x"], td)
    b = to_dev(p["b"], td)
    a = to_dev(p["a"], td)
    zi = to_dev(p["zi"], td)
    gy = to_dev(p["gy"], td)
    gzf = to_dev(p["gzf"], td)
    Bsz, T = x.shape
    M = b.shape[-1] - 1
    if coef_mode is None:
        coef_mode = B.IIR_COEF_SHARED if b.dim() == 1 else B.IIR_COEF_PER_SEQ
    desc = B.make_desc(Bsz, T, M, p["form"], td, coef_mode, flags=flags)
    desc_b = B.make_desc(Bsz, T, M, p["form"], td, coef_mode, flags=flags if flags_bwd is None else flags_bwd)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    tape = torch.empty(tb, dtype=torch.uint8, device="cuda")
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    y = torch.full_like(x, float("nan"))
    zf = torch.full((Bsz, M), float("nan"), dtype=td, device="cuda") if "zf" in want else None
    gx = torch.full_like(x, float("nan")) if "gx" in want else None
    gb = torch.full_like(b, float("nan")) if "gb" in want else None
    ga = torch.full_like(a, float("nan")) if "ga" in want else None
    gzi = torch.full((Bsz, M), float("nan"), dtype=td, device="cuda") if "gzi" in want else None
    for _ in range(repeat):
        B.iir_forward(desc, b, a, x, zi, y, zf, tape, tb, ws, wb, stream)
        B.iir_backward(desc_b, gy, gzf, b, a, x, y, zi, tape, tb, gx, gb, ga, gzi, ws, wb, stream)
    torch.cuda.synchronize()
    out = {"y": y, "zf": zf, "gx": gx, "gb": gb, "ga": ga, "gzi": gzi}
    return {k: (None if v is None else v.double().cpu().numpy()) for k, v in out.items()}


def run_lti_oracle(p, seqs=None):
    form = 1 if p["form"] == "tdf" else 0
    sl = slice(None) if seqs is None else seqs
    shared = p["b"].ndim == 1
    b = p["b"] if shared else p["b"][sl]
    a = p["a"] if shared else p["a"][sl]
    return oracle.lti(form, b, a, p["x"][sl], None if p["zi"] is None else p["zi"][sl], p["gy"][sl],
                      None if p["gzf"] is None else p["gzf"][sl])


def compare(g, o, tol, keys=("y", "zf", "gx", "gb", "ga", "gzi"), seqs=None):
    """Per-tensor normalised errors; with `seqs` only those sequences are
    compared (shared-coefficient gradients are then skipped: they sum over
    the whole batch)."""
    errs = {}
    for k in keys:
        if g.get(k) is None:
            continue
        gg = g[k]
        if seqs is not None:
            if k in ("gb", "ga") and gg.ndim == 1:
                continue
            gg = gg[seqs]
        errs[k] = nrm_err(gg, o[k])
    bad = {k: v for k, v in errs.items() if not (v <= tol)}
    return errs, bad
