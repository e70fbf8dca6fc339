"""Robustness of the CUDA path (VERDICT r1 "missing" #6):
NULL grad_y, NaN / inf inputs propagate (no hang, no trap, no look-back timeout),
back-to-back backward calls on one IIR_FLAG_WS_READY workspace, a caller kernel
writing grad_y right before iir_backward, and a negative control showing that
the parity measure flags a wrong result."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_14390_b200 import _binding as B
from paper_2511_14390_b200 import inputs

from gpu_util import TOL, compare, nrm_err, run_lti_gpu, run_lti_oracle, to_dev

pytestmark = pytest.mark.gpu


def _bufs(p, flags=0):
    td = torch.float32 if p["dtype"] == "f32" else torch.float64
    if p["form"] == "tdf" and p["dtype"] == "f32":
        flags |= B.IIR_FLAG_ENGINE_V2                  # the round-2 engine (the default only from order 6)
    x, b, a, zi, gy, gzf = (to_dev(p[k], td) for k in ("x", "b", "a", "zi", "gy", "gzf"))
    Bsz, T = x.shape
    M = b.shape[-1] - 1
    desc = B.make_desc(Bsz, T, M, p["form"], td, B.IIR_COEF_SHARED if b.dim() == 1 else B.IIR_COEF_PER_SEQ,
                       flags=flags)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    tape = torch.empty(tb, dtype=torch.uint8, device="cuda")
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    return dict(x=x, b=b, a=a, zi=zi, gy=gy, gzf=gzf, desc=desc, tb=tb, wb=wb, tape=tape, ws=ws, M=M)


def _fwd_bwd(s, gy="gy", x=None):
    x = s["x"] if x is None else x
    y = torch.empty_like(x)
    zf = torch.empty_like(s["zi"])
    gx = torch.empty_like(x)
    gb, ga, gzi = torch.empty_like(s["b"]), torch.empty_like(s["a"]), torch.empty_like(s["zi"])
    B.iir_forward(s["desc"], s["b"], s["a"], x, s["zi"], y, zf, s["tape"], s["tb"], s["ws"], s["wb"])
    B.iir_backward(s["desc"], None if gy is None else s[gy], s["gzf"], s["b"], s["a"], x, y, s["zi"], s["tape"],
                   s["tb"], gx, gb, ga, gzi, s["ws"], s["wb"])
    torch.cuda.synchronize()
    return dict(y=y, zf=zf, gx=gx, gb=gb, ga=ga, gzi=gzi)


@pytest.mark.parametrize("form,dtype,M", [("tdf", "f32", 8), ("tdf", "f32", 2), ("df", "f32", 3), ("tdf", "f64", 2)])
def test_null_grad_y(form, dtype, M):
    """grad_y = NULL means zeros (include/iirgrad.h): only grad_zf drives the adjoint."""
    p = inputs.lti_problem(8100 + M, form=form, order=M, batch=3, length=3 * 2048 + 19, dtype=dtype,
                           angles="spread")
    s = _bufs(p)
    g = _fwd_bwd(s, gy=None)
    q = dict(p, gy=np.zeros_like(p["gy"]))
    o = run_lti_oracle(q)
    errs, bad = compare({k: v.double().cpu().numpy() for k, v in g.items()}, o, TOL[dtype])
    assert not bad, errs


def test_null_grad_y_per_sample():
    p = inputs.tv_allpole_problem(8200, batch=2, length=3000, order=8, dtype="f32", hop=128)
    q = {k: None if p[k] is None else np.asarray(p[k], np.float64) for k in ("a", "x", "zi", "gy", "gzf")}
    td = torch.float32
    dev = lambda v: torch.tensor(v, dtype=td, device="cuda")
    a, x, zi, gzf = dev(q["a"]), dev(q["x"]), dev(q["zi"]), dev(q["gzf"])
    desc = B.make_desc(2, 3000, 8, "df", td, B.IIR_COEF_PER_SAMPLE)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    tape = torch.empty(tb, dtype=torch.uint8, device="cuda")
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    y, zf, gx, ga, gzi = torch.empty_like(x), torch.empty_like(zi), torch.empty_like(x), torch.empty_like(a), \
        torch.empty_like(zi)
    B.iir_forward(desc, None, a, x, zi, y, zf, tape, tb, ws, wb)
    B.iir_backward(desc, None, gzf, None, a, None, y, zi, tape, tb, gx, None, ga, gzi, ws, wb)
    torch.cuda.synchronize()
    o = oracle.tv_allpole(q["a"], q["x"], q["zi"], np.zeros_like(q["gy"]), q["gzf"])
    for k, t in (("y", y), ("gx", gx), ("ga", ga), ("gzi", gzi)):
        assert nrm_err(t.double().cpu().numpy(), o[k]) < 1e-4, k


@pytest.mark.parametrize("form,dtype,M", [("tdf", "f32", 8), ("tdf", "f32", 4), ("df", "f32", 3), ("tdf", "f64", 2)])
@pytest.mark.parametrize("bad", [float("nan"), float("inf"), -float("nan")])
def test_nan_inf_propagate(form, dtype, M, bad):
    """A NaN / inf in one sequence's x propagates forward in time in that sequence
    only; the call completes (no hang, no trap, no look-back timeout) and the other
    sequences are unaffected.  -nan has the sign bit set (the bit pattern nearest the
    look-back sentinel)."""
    T = 5 * 2048 + 100
    p = inputs.lti_problem(8300 + M, form=form, order=M, batch=3, length=T, dtype=dtype, angles="spread")
    s = _bufs(p, flags=B.IIR_FLAG_WS_READY)
    B.iir_workspace_init(s["desc"], s["ws"], s["wb"])
    clean = _fwd_bwd(s)
    n0 = 3 * 2048 + 7
    x2 = s["x"].clone()
    x2[1, n0] = bad
    g = _fwd_bwd(s, x=x2)
    B.iir_check_workspace(s["desc"], s["ws"], s["wb"])          # raises if a look-back timed out
    y = g["y"].double().cpu().numpy()
    yc = clean["y"].double().cpu().numpy()
    assert np.array_equal(y[[0, 2]], yc[[0, 2]])                 # other sequences bitwise unaffected
    assert np.array_equal(y[1, :n0], yc[1, :n0])                 # the past is unaffected
    assert not np.isfinite(y[1, n0])                            # the bad sample reaches the output
    assert np.all(~np.isfinite(y[1, n0 + M + 1:]) | (np.abs(y[1, n0 + M + 1:]) > 1e30))
    # a clean call after the bad one: the workspace is intact
    g2 = _fwd_bwd(s)
    for k in ("y", "gx", "gb", "ga"):
        assert torch.equal(g2[k], clean[k]), k


@pytest.mark.parametrize("form", ["tdf", "df"])
def test_nan_in_grad_y_propagates_backward(form):
    T = 4 * 2048 + 33
    p = inputs.lti_problem(8400, form=form, order=4, batch=2, length=T, dtype="f32", angles="spread")
    s = _bufs(p)
    clean = _fwd_bwd(s)
    s["gy2"] = s["gy"].clone()
    s["gy2"][0, 5000] = float("nan")
    g = _fwd_bwd(s, gy="gy2")
    gx = g["gx"].double().cpu().numpy()
    gxc = clean["gx"].double().cpu().numpy()
    assert np.array_equal(gx[1], gxc[1])
    assert np.array_equal(gx[0, 5001:], gxc[0, 5001:])           # the adjoint runs backwards in time
    assert np.isnan(gx[0, 5000])
    assert not np.all(np.isfinite(g["ga"].cpu().numpy()))       # shared-coefficient gradients see it


@pytest.mark.parametrize("M", [2, 8])
def test_ws_ready_back_to_back_backward(M):
    """two backward calls in a row on one IIR_FLAG_WS_READY workspace (no
    memset in between) and a caller kernel writing grad_y immediately before
    iir_backward on the same stream."""
    p = inputs.lti_problem(8500 + M, form="tdf", order=M, batch=4, length=6 * 2048 + 5, dtype="f32",
                           angles="spread")
    s = _bufs(p, flags=B.IIR_FLAG_WS_READY)
    B.iir_workspace_init(s["desc"], s["ws"], s["wb"])
    o = run_lti_oracle(p)
    y, zf = torch.empty_like(s["x"]), torch.empty_like(s["zi"])
    B.iir_forward(s["desc"], s["b"], s["a"], s["x"], s["zi"], y, zf, s["tape"], s["tb"], s["ws"], s["wb"])
    for rep in range(3):
        gy = torch.mul(s["gy"], 1.0)          # a caller kernel producing grad_y right before the call
        gx, gzi = torch.empty_like(s["x"]), torch.empty_like(s["zi"])
        gb, ga = torch.empty_like(s["b"]), torch.empty_like(s["a"])
        B.iir_backward(s["desc"], gy, s["gzf"], s["b"], s["a"], s["x"], y, s["zi"], s["tape"], s["tb"], gx, gb,
                       ga, gzi, s["ws"], s["wb"])
        torch.cuda.synchronize()
        for k, t in (("gx", gx), ("gb", gb), ("ga", ga), ("gzi", gzi)):
            assert nrm_err(t.double().cpu().numpy(), o[k]) < 1e-4, (rep, k)
    B.iir_check_workspace(s["desc"], s["ws"], s["wb"])


def test_negative_control_flags_wrong_results():
    """The parity measure has power: a result off by 10x the gate in ONE element, or
    computed with a coefficient perturbed in its 4th significant digit, fails it."""
    p = inputs.lti_problem(8600, form="tdf", order=4, batch=4, length=3 * 2048, dtype="f32", angles="spread")
    o = run_lti_oracle(p)
    g = run_lti_gpu(p, flags=B.IIR_FLAG_ENGINE_V2)
    errs, bad = compare(g, o, TOL["f32"])
    assert not bad, errs                                         # the real result passes
    for k in ("y", "gx", "gb", "ga", "gzi", "zf"):
        h = {kk: v.copy() for kk, v in g.items()}
        flat = h[k].reshape(-1)
        flat[len(flat) // 2] += 10 * TOL["f32"] * np.sqrt(np.mean(o[k] ** 2))
        _, bad = compare(h, o, TOL["f32"])
        assert k in bad, f"a corrupted {k} passed the gate"
    q = dict(p, a=p["a"].copy())
    q["a"][1] *= 1.0 + 1e-3                                      # a wrong filter on the GPU side
    gw = run_lti_gpu(q, flags=B.IIR_FLAG_ENGINE_V2)
    _, bad = compare(gw, o, TOL["f32"])
    assert {"y", "gx"} <= set(bad), bad


def test_config5_shard_bitwise_deterministic():
    """Same inputs, same descriptor -> bitwise-identical outputs (fixed reduction order,
    no floating-point atomics), although the persistent warps take tiles by ticket."""
    p = inputs.lti_problem(8700, form="tdf", order=8, batch=64, length=1 << 16, dtype="f32", angles="spread")
    g1 = run_lti_gpu(p)
    g2 = run_lti_gpu(p)
    for k in g1:
        assert np.array_equal(g1[k], g2[k]), k


def test_check_workspace_clean():
    p = inputs.lti_problem(8800, form="tdf", order=3, batch=2, length=5000, dtype="f32")
    s = _bufs(p)
    _fwd_bwd(s)
    B.iir_check_workspace(s["desc"], s["ws"], s["wb"])
