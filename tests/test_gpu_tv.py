"""GPU parity of the per-sample (time-varying) all-pole DF path (SURVEY §8(a)
row a9, config 3) against the fp64 oracle (orc_tv_allpole) on the same
dtype-rounded inputs; gate: fp32 1e-4, fp64 1e-10 of max|err| / rms."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_14390_b200 import _binding as B
from paper_2511_14390_b200 import inputs

from gpu_util import TOL, nrm_err

pytestmark = pytest.mark.gpu


def run_tv_gpu(p, dtype):
    td = torch.float32 if dtype == "f32" else torch.float64
    dev = lambda t: None if t is None else torch.as_tensor(np.asarray(t), dtype=torch.float64).to(td).cuda()
    a, x, zi, gy, gzf = map(dev, (p["a"], p["x"], p["zi"], p["gy"], p["gzf"]))
    Bsz, T = x.shape
    M = a.shape[-1]
    desc = B.make_desc(Bsz, T, M, "df", td, B.IIR_COEF_PER_SAMPLE)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    assert tb > 0 and wb > 0
    tape = torch.empty(tb, dtype=torch.uint8, device="cuda")
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    y = torch.full_like(x, float("nan"))
    zf = torch.full((Bsz, M), float("nan"), dtype=td, device="cuda")
    gx = torch.full_like(x, float("nan"))
    ga = torch.full_like(a, float("nan"))
    gzi = torch.full((Bsz, M), float("nan"), dtype=td, device="cuda")
    B.iir_forward(desc, None, a, x, zi, y, zf, tape, tb, ws, wb)
    B.iir_backward(desc, gy, gzf, None, a, None, y, zi, tape, tb, gx, None, ga, gzi, ws, wb)
    torch.cuda.synchronize()
    f = lambda t: t.double().cpu().numpy()
    return dict(y=f(y), zf=f(zf), gx=f(gx), ga=f(ga), gzi=f(gzi))


def np_problem(p, dtype):
    t = np.float32 if dtype == "f32" else np.float64
    c = lambda v: None if v is None else np.asarray(v.numpy() if torch.is_tensor(v) else v).astype(t).astype(np.float64)
    return {k: c(p[k]) for k in ("a", "x", "zi", "gy", "gzf")}


def check(p, dtype, tol=None):
    tol = TOL[dtype] if tol is None else tol
    q = np_problem(p, dtype)
    g = run_tv_gpu(q, dtype)
    o = oracle.tv_allpole(q["a"], q["x"], q["zi"], q["gy"], q["gzf"])
    errs = {k: nrm_err(g[k], o[k]) for k in ("y", "zf", "gx", "ga", "gzi")}
    bad = {k: v for k, v in errs.items() if not v <= tol}
    assert not bad, f"errors {errs} exceed {tol}"
    return errs


def test_config3_shape_lpc24_fp32():
    """Config-3 recipe (LPC order 24, per-sample coefficients) on 4 of the 32
    sequences at full length 2^18."""
    p = inputs.tv_allpole_problem(1003, batch=4, length=1 << 18, order=24, dtype="f32")
    check(p, "f32")


@pytest.mark.parametrize("M", [1, 2, 3, 4, 8, 9, 11, 12, 13, 16, 17, 18, 21, 24, 25, 27, 30, 31])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_orders(M, dtype):
    p = inputs.tv_allpole_problem(2100 + M, batch=3, length=5 * 512 + 37, order=M, dtype=dtype, hop=128)
    check(p, dtype)


@pytest.mark.parametrize("T", [1, 2, 5, 23, 24, 25, 511, 512, 513, 1024, 1500])
def test_edge_lengths(T):
    p = inputs.tv_allpole_problem(2200 + T, batch=2, length=T, order=24, dtype="f64", hop=64)
    check(p, "f64")


def test_no_initial_conditions():
    p = inputs.tv_allpole_problem(2300, batch=2, length=4000, order=8, dtype="f32", zi=False, gzf=False)
    check(p, "f32")


def test_every_order_up_to_32_supported_33_rejected():
    """Every per-sample order 1..32 is compiled (orders up to 32 for the
    per-sample path; the Phi kernel runs a second column block at 32); 33 is rejected
    before any launch."""
    for M in range(1, 33):
        assert B.iir_tape_bytes(B.make_desc(1, 100, M, "df", torch.float32, B.IIR_COEF_PER_SAMPLE)) > 0, M
    assert B.iir_tape_bytes(B.make_desc(1, 100, 33, "df", torch.float32, B.IIR_COEF_PER_SAMPLE)) == 0


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("M", [9, 18, 31, 32])
def test_lpc_orders(M, dtype):
    """LPC orders the round-1 build rejected (9, 18) and the two column-block edge (31, 32)
    of the segment-transition kernel, several segments and a ragged tail."""
    p = inputs.tv_allpole_problem(2500 + M, batch=3, length=3 * 512 + 77, order=M, dtype=dtype)
    check(p, dtype)


def test_autograd_allpole_tv():
    from paper_2511_14390_b200 import allpole_tv
    p = inputs.tv_allpole_problem(2400, batch=2, length=3000, order=6, dtype="f64", hop=100)
    q = np_problem(p, "f64")
    T = lambda v: torch.tensor(v, dtype=torch.float64, device="cuda", requires_grad=True)
    a, x, zi = T(q["a"]), T(q["x"]), T(q["zi"])
    y, zf = allpole_tv(x, a, zi, return_zf=True)
    (y * torch.tensor(q["gy"], device="cuda")).sum().add((zf * torch.tensor(q["gzf"], device="cuda")).sum()).backward()
    o = oracle.tv_allpole(q["a"], q["x"], q["zi"], q["gy"], q["gzf"])
    assert nrm_err(x.grad.cpu().numpy(), o["gx"]) < 1e-10
    assert nrm_err(a.grad.cpu().numpy(), o["ga"]) < 1e-10
    assert nrm_err(zi.grad.cpu().numpy(), o["gzi"]) < 1e-10


def test_config3_full_batch_fp32():
    """Config 3 at its full size: all 32 sequences x 2^18 samples, LPC order 24, every
    output element against the oracle (was 4 of 32)."""
    c = inputs.CONFIGS["c3"]
    p = inputs.tv_allpole_problem(1003, batch=c["batch"], length=c["length"], order=c["order"], dtype="f32")
    check(p, "f32")


def test_config3_shape_fp64_exact_algorithm():
    """Same recipe in fp64: isolates the algorithm from fp32 rounding."""
    p = inputs.tv_allpole_problem(1003, batch=2, length=1 << 18, order=24, dtype="f64")
    check(p, "f64")
