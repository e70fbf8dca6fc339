"""Small invocations of every kernel family through the C ABI, for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize_cases.py.  Exits non-zero on a
parity failure (checked against the fp64 oracle) so a sanitizer run also checks results."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402
from paper_2511_14390_b200 import _binding as B  # noqa: E402
from paper_2511_14390_b200 import inputs  # noqa: E402
from gpu_util import compare, run_lti_gpu, run_lti_oracle, nrm_err  # noqa: E402


def lti(seed, form, M, dtype, batch, T, coef="shared", flags=0):
    p = inputs.lti_problem(seed, form=form, order=M, batch=batch, length=T, dtype=dtype, coef=coef, angles="spread")
    g = run_lti_gpu(p, flags=flags)
    errs, bad = compare(g, run_lti_oracle(p), 1e-4 if dtype == "f32" else 1e-10)
    print(f"lti {form} M={M} {dtype} B={batch} T={T} {coef} flags={flags}: {errs}", flush=True)
    return not bad


def tv(seed, M, fir):
    p = inputs.tv_df_problem(seed, batch=2, length=1500, order=M, dtype="f32", hop=128)
    q = {k: None if p[k] is None else np.asarray(p[k], np.float64) for k in ("b", "a", "x", "zi", "gy", "gzf")}
    dev = lambda v: torch.tensor(v, dtype=torch.float32, device="cuda")
    b_, a_, x_, zi_, gy_, gzf_ = (dev(q[k]) for k in ("b", "a", "x", "zi", "gy", "gzf"))
    desc = B.make_desc(2, 1500, M, "df", torch.float32, B.IIR_COEF_PER_SAMPLE,
                       flags=B.IIR_FLAG_PER_SAMPLE_B if fir else 0)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    tape = torch.empty(tb, dtype=torch.uint8, device="cuda")
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    y, gx, ga = torch.empty_like(x_), torch.empty_like(x_), torch.empty_like(a_)
    zf, gzi = torch.empty_like(zi_), torch.empty_like(zi_)
    gb = torch.empty_like(b_) if fir else None
    B.iir_forward(desc, b_ if fir else None, a_, x_, zi_, y, zf, tape, tb, ws, wb)
    B.iir_backward(desc, gy_, gzf_, b_ if fir else None, a_, None, y, zi_, tape, tb, gx, gb, ga, gzi, ws, wb)
    torch.cuda.synchronize()
    o = oracle.tv_df(q["b"], q["a"], q["x"], q["zi"], q["gy"], q["gzf"]) if fir else \
        oracle.tv_allpole(q["a"], q["x"], q["zi"], q["gy"], q["gzf"])
    got = dict(y=y, zf=zf, gx=gx, ga=ga, gzi=gzi, **({"gb": gb} if fir else {}))
    errs = {k: nrm_err(t.double().cpu().numpy(), o[k]) for k, t in got.items()}
    print(f"tv M={M} fir={fir}: {errs}", flush=True)
    return all(v < 1e-4 for v in errs.values())


def main():
    torch.cuda.set_device(0)
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    ok = True
    if which in ("all", "lti"):
        ok &= lti(1, "tdf", 8, "f32", 3, 3 * 2048 + 76)          # round-2 engine, ragged tail
        ok &= lti(2, "tdf", 2, "f32", 2, 40 * 2048)              # round-2 engine, two look-back levels
        ok &= lti(3, "tdf", 3, "f32", 3, 2 * 2048 + 5, coef="per_seq")   # unaligned length: element copies
        ok &= lti(4, "tdf", 4, "f32", 2, 3 * 4096 + 8, flags=B.IIR_FLAG_LEGACY_LTI)
        ok &= lti(5, "df", 3, "f32", 2, 3 * 4096 + 9)
        ok &= lti(6, "tdf", 2, "f64", 1, 4096)
    if which in ("all", "tv"):
        ok &= tv(7, 6, False)
        ok &= tv(8, 6, True)
    print("sanitize cases:", "ok" if ok else "PARITY FAILURE", flush=True)
    sys.exit(0 if ok else 3)


if __name__ == "__main__":
    main()
