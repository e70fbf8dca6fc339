"""GPU parity of the bare recurrence v(n+1) = A v(n) + z(n) (form IIR_SS, SURVEY
§8(f) f1, Listing 1) against oracle.recurrence, through the C ABI.
Sizes span several tiles and a ragged tail; gates as for the filters (R13)."""
import numpy as np
import pytest
import torch

import oracle
from paper_2511_14390_b200 import _binding as B
from paper_2511_14390_b200 import inputs

from gpu_util import TOL, nrm_err, to_dev

pytestmark = pytest.mark.gpu


def run_gpu(p, want_v0_grad=True, flags=0):
    td = torch.float32 if p["dtype"] == "f32" else torch.float64
    A, z, gv = to_dev(p["A"], td), to_dev(p["z"], td), to_dev(p["gv"], td)
    v0 = to_dev(p["v0"], td)
    Bsz, N, M = z.shape
    mode = B.IIR_COEF_SHARED if A.dim() == 2 else B.IIR_COEF_PER_SEQ
    desc = B.make_desc(Bsz, N, M, "ss", td, mode, flags=flags)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    tape = torch.empty(tb, dtype=torch.uint8, device="cuda")
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    v = torch.full_like(z, float("nan"))
    gz = torch.full_like(z, float("nan"))
    gA = torch.full_like(A, float("nan"))
    gv0 = torch.full_like(v0, float("nan")) if (v0 is not None and want_v0_grad) else None
    B.iir_forward(desc, None, A, z, v0, v, None, tape, tb, ws, wb)
    B.iir_backward(desc, gv, None, None, A, None, v, v0, tape, tb, gz, None, gA, gv0, ws, wb)
    torch.cuda.synchronize()
    out = dict(v=v, gz=gz, gA=gA, gv0=gv0)
    return {k: (None if t is None else t.double().cpu().numpy()) for k, t in out.items()}


def run_oracle(p):
    Bsz, N, M = p["z"].shape
    shared = p["A"].ndim == 2
    res = {"v": [], "gz": [], "gv0": [], "gA": []}
    for b in range(Bsz):
        A = p["A"] if shared else p["A"][b]
        v0 = np.zeros(M) if p["v0"] is None else p["v0"][b]
        o = oracle.recurrence(A, v0, p["z"][b], p["gv"][b])
        for k in res:
            res[k].append(o[k])
    out = {k: np.stack(v) for k, v in res.items()}
    if shared:
        out["gA"] = out["gA"].sum(axis=0)
    return out


def check(p, flags=0):
    g, o = run_gpu(p, flags=flags), run_oracle(p)
    tol = TOL[p["dtype"]]
    for k in ("v", "gz", "gA", "gv0"):
        if g[k] is None:
            continue
        e = nrm_err(g[k], o[k])
        assert e <= tol, f"{k}: normalised error {e:.3e} > {tol:g}"


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("M", [1, 2, 3, 4])
def test_orders_dtypes(dtype, M):
    check(inputs.rec_problem(9000 + M, batch=3, length=3 * 4096 + 77, order=M, dtype=dtype))


@pytest.mark.parametrize("N", [1, 2, 3, 31, 33, 2047, 4096, 4097, 10001])
def test_lengths(N):
    check(inputs.rec_problem(9100 + N, batch=2, length=N, order=2, dtype="f32"))


def test_per_sequence_A_and_zero_v0():
    check(inputs.rec_problem(9200, batch=4, length=9000, order=2, dtype="f32", coef="per_seq"))
    check(inputs.rec_problem(9201, batch=2, length=5000, order=3, dtype="f64", v0=False))


def test_long_sequence_multi_level_lookback():
    # 2^20 samples: 256 tiles of 4096 -> two look-back levels (the paper's longest N)
    p = inputs.rec_problem(9300, batch=1, length=1 << 20, order=2, dtype="f32", r_hi=0.999)
    check(p)


def test_autograd_matches_oracle():
    from paper_2511_14390_b200 import matrix_recurrence
    p = inputs.rec_problem(9400, batch=2, length=5000, order=2, dtype="f64")
    A = torch.tensor(p["A"], device="cuda", requires_grad=True)
    v0 = torch.tensor(p["v0"], device="cuda", requires_grad=True)
    z = torch.tensor(p["z"], device="cuda", requires_grad=True)
    v = matrix_recurrence(A, v0, z)
    (v * torch.tensor(p["gv"], device="cuda")).sum().backward()
    o = run_oracle(p)
    assert nrm_err(v.detach().cpu().numpy(), o["v"]) <= 1e-10
    assert nrm_err(z.grad.cpu().numpy(), o["gz"]) <= 1e-10
    assert nrm_err(A.grad.cpu().numpy(), o["gA"]) <= 1e-10
    assert nrm_err(v0.grad.cpu().numpy(), o["gv0"]) <= 1e-10
