"""GPU parity of the general time-varying TDF-II path (form IIR_TDF2 with
IIR_FLAG_PER_SAMPLE_B, reading R20: the TDF realisation of
PAPER.md:67-68 at every sample) against the fp64 oracle orc_tv_tdf on the same
dtype-rounded inputs; gate: fp32 1e-4, fp64 1e-10 of max|err| / rms per output tensor
(y, zf, grad_x, grad_b, grad_a, grad_zi)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_14390_b200 import _binding as B
from paper_2511_14390_b200 import inputs

from gpu_util import TOL, nrm_err
from test_gpu_tvdf import rounded

pytestmark = pytest.mark.gpu


def run(q, dtype, want=("y", "zf", "gx", "gb", "ga", "gzi")):
    td = torch.float32 if dtype == "f32" else torch.float64
    dev = lambda t: None if t is None else torch.as_tensor(np.asarray(t), dtype=torch.float64).to(td).cuda()
    b, a, x, zi, gy, gzf = map(dev, (q["b"], q["a"], q["x"], q["zi"], q["gy"], q["gzf"]))
    Bsz, T = x.shape
    M = a.shape[-1]
    desc = B.make_desc(Bsz, T, M, "tdf", td, B.IIR_COEF_PER_SAMPLE, flags=B.IIR_FLAG_PER_SAMPLE_B)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    assert tb > 0 and wb > 0
    tape = torch.empty(tb, dtype=torch.uint8, device="cuda")
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    nan = lambda *s: torch.full(s, float("nan"), dtype=td, device="cuda")
    y = nan(Bsz, T)
    out = dict(zf=nan(Bsz, M), gx=nan(Bsz, T), gb=nan(Bsz, T, M + 1), ga=nan(Bsz, T, M), gzi=nan(Bsz, M))
    out = {k: (v if k in want else None) for k, v in out.items()}
    B.iir_forward(desc, b, a, x, zi, y, out["zf"], tape, tb, ws, wb)
    B.iir_backward(desc, gy, gzf, b, a, x, y, zi, tape, tb, out["gx"], out["gb"], out["ga"], out["gzi"], ws, wb)
    torch.cuda.synchronize()
    f = lambda t: None if t is None else t.double().cpu().numpy()
    return dict(y=f(y), **{k: f(v) for k, v in out.items()})


def check(p, dtype, tol=None, want=("y", "zf", "gx", "gb", "ga", "gzi")):
    tol = TOL[dtype] if tol is None else tol
    q = rounded(p, dtype)
    g = run(q, dtype, want)
    o = oracle.tv_tdf(q["b"], q["a"], q["x"], q["zi"], q["gy"], q["gzf"])
    errs = {k: nrm_err(g[k], o[k]) for k in want}
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"errors {errs} exceed {tol}"
    return errs


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("M", [1, 2, 4, 8, 9, 24, 32])
def test_orders_dtypes(dtype, M):
    p = inputs.tv_df_problem(35000 + M, batch=3, length=3 * 512 + 37, order=M, dtype=dtype, hop=128)
    check(p, dtype)


@pytest.mark.parametrize("T", [1, 2, 3, 5, 23, 24, 25, 511, 512, 513, 1500])
def test_edge_lengths(T):
    """Lengths below the order (zi reaches zf directly), at and around segment edges."""
    p = inputs.tv_df_problem(36000 + T, batch=2, length=T, order=24, dtype="f64", hop=64)
    check(p, "f64")


@pytest.mark.parametrize("zi,gzf", [(False, False), (True, False), (False, True)])
def test_initial_condition_paths(zi, gzf):
    p = inputs.tv_df_problem(37000, batch=2, length=3000, order=8, dtype="f32", zi=zi, gzf=gzf)
    check(p, "f32")


def test_null_optional_outputs():
    p = inputs.tv_df_problem(37100, batch=2, length=2000, order=4, dtype="f32")
    check(p, "f32", want=("y", "gx"))


def test_constant_rows_equal_lti_tdf_engine():
    """Constant rows: the per-sample TDF equals the LTI TDF path of the library (scipy's lfilter)."""
    p = inputs.tv_df_problem(37200, batch=2, length=5000, order=3, dtype="f64")
    p["b"][:] = p["b"][:, :1, :]
    p["a"][:] = p["a"][:, :1, :]
    q = rounded(p, "f64")
    g = run(q, "f64")
    from gpu_util import run_lti_gpu
    lp = dict(form="tdf", b=q["b"][:, 0], a=np.concatenate([np.ones((2, 1)), q["a"][:, 0]], axis=1), x=q["x"],
              gy=q["gy"], zi=q["zi"], gzf=q["gzf"], dtype="f64")
    l = run_lti_gpu(lp)
    for k in ("y", "zf", "gx", "gzi"):
        assert nrm_err(g[k], l[k]) < 1e-10, k
    assert nrm_err(g["gb"].sum(axis=1), l["gb"]) < 1e-10


def test_config3_shape_tdf_fp32():
    """Config-3 shape (order 24, per-sample rows, 2^18 samples), 4 sequences."""
    p = inputs.tv_df_problem(1003, batch=4, length=1 << 18, order=24, dtype="f32")
    check(p, "f32")


def test_autograd_function_matches_oracle():
    from paper_2511_14390_b200 import lfilter_tv
    p = inputs.tv_df_problem(38000, batch=2, length=3000, order=6, dtype="f32")
    q = rounded(p, "f32")
    dev = lambda v: torch.tensor(v, dtype=torch.float32, device="cuda", requires_grad=True)
    x, b, a, zi = dev(q["x"]), dev(q["b"]), dev(q["a"]), dev(q["zi"])
    y, zf = lfilter_tv(x, b, a, zi=zi, return_zf=True, form="tdf")
    L = (y * torch.tensor(q["gy"], dtype=torch.float32, device="cuda")).sum() + \
        (zf * torch.tensor(q["gzf"], dtype=torch.float32, device="cuda")).sum()
    L.backward()
    o = oracle.tv_tdf(q["b"], q["a"], q["x"], q["zi"], q["gy"], q["gzf"])
    for k, t in (("y", y.detach()), ("zf", zf.detach()), ("gx", x.grad), ("gb", b.grad), ("ga", a.grad),
                 ("gzi", zi.grad)):
        assert nrm_err(t.double().cpu().numpy(), o[k]) < 1e-4, k


def test_gradcheck_fp64_tiny():
    from paper_2511_14390_b200 import lfilter_tv
    torch.manual_seed(0)
    mk = lambda *s: (0.2 * torch.randn(*s, dtype=torch.float64, device="cuda")).requires_grad_(True)
    x, b, a, zi = mk(2, 19), mk(2, 19, 4), mk(2, 19, 3), mk(2, 3)
    f = lambda x, b, a, zi: lfilter_tv(x, b, a, zi=zi, return_zf=True, form="tdf")
    assert torch.autograd.gradcheck(f, (x, b, a, zi), eps=1e-6, atol=1e-8, rtol=1e-6)


def test_gradients_without_grad_x_output():
    """grad_x = NULL (the FIR adjoint then writes into scratch), grad_zf given: the other
    gradients are unchanged."""
    p = inputs.tv_df_problem(37300, batch=2, length=1300, order=5, dtype="f64")
    check(p, "f64", want=("y", "zf", "gb", "ga", "gzi"))
