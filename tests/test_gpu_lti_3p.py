"""GPU parity of the LTI path's three-phase schedule (IIR_FLAG_THREE_PHASE:
lti_red_kernel -> lti_cscan_kernel -> emit from precomputed carries) against
the fp64 oracle, and its agreement with the single-pass schedule.  Same gate
as test_gpu_lti.py (north star): fp32 1e-4, fp64 1e-10 of max|gpu - oracle| /
rms(oracle) per output tensor.  The carry scan works in runs of 32 tiles per
thread, 1024 per warp and passes of 4096 tiles: the tile counts below straddle
those boundaries."""
import numpy as np
import pytest
import torch

from paper_2511_14390_b200 import _binding as B
from paper_2511_14390_b200 import inputs

from gpu_util import TOL, compare, nrm_err, run_lti_gpu, run_lti_oracle

pytestmark = pytest.mark.gpu

P3 = B.IIR_FLAG_THREE_PHASE
P1 = B.IIR_FLAG_SINGLE_PASS
TS = {"f32": 4096, "f64": 2048}


def tile(dtype, M):
    return TS[dtype] * (2 if M >= 4 else 1)


def check(p, flags=P3, tol=None, seqs=None, **kw):
    tol = TOL[p["dtype"]] if tol is None else tol
    g = run_lti_gpu(p, flags=flags, **kw)
    o = run_lti_oracle(p, seqs)
    errs, bad = compare(g, o, tol, seqs=seqs)
    assert not bad, f"errors {errs} exceed {tol}"
    return g


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("M", [1, 2, 3, 4, 5, 6, 7, 8])
def test_orders_forms_dtypes(dtype, form, M):
    p = inputs.lti_problem(12000 + M, form=form, order=M, batch=3, length=3 * tile(dtype, M) + 77, dtype=dtype,
                           angles="spread")
    check(p)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("T", [1, 2, 3, 5, 31, 33, 4095, 4096, 4097, 2049, 8191, 10007])
def test_edge_lengths(dtype, form, T):
    p = inputs.lti_problem(13000 + T, form=form, order=3, batch=2, length=T, dtype=dtype)
    check(p)


@pytest.mark.parametrize("ntiles", [1, 2, 31, 32, 33, 63, 64, 65, 1023, 1024, 1025, 2047, 4095, 4096, 4097, 5000])
def test_carry_scan_run_warp_pass_boundaries(ntiles):
    """One sequence of `ntiles` tiles (M = 2, 4096-sample tiles), ragged tail."""
    p = inputs.lti_problem(14000 + ntiles, form="tdf", order=2, batch=1, length=ntiles * 4096 - 5, dtype="f32",
                           angles="spread")
    check(p)


@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("M", [4, 8])
def test_long_sequence_high_order(form, M):
    """Several thousand tiles of order 4 / 8 (runs and passes at the longer 8192-sample tiles)."""
    p = inputs.lti_problem(14500 + M, form=form, order=M, batch=1, length=4100 * 8192 + 3, dtype="f32",
                           angles="spread")
    check(p)


@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("zi,gzf", [(False, False), (True, False), (False, True), (True, True)])
def test_initial_condition_paths(form, zi, gzf):
    p = inputs.lti_problem(15000, form=form, order=4, batch=5, length=40000, dtype="f32", zi=zi, gzf=gzf,
                           angles="spread")
    check(p)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("form", ["tdf", "df"])
def test_per_sequence_coefficients(dtype, form):
    p = inputs.lti_problem(16000, form=form, order=4, batch=7, length=5 * TS[dtype] + 5, dtype=dtype,
                           coef="per_seq", angles="spread")
    check(p)


@pytest.mark.parametrize("form", ["tdf", "df"])
def test_unnormalised_a0(form):
    p = inputs.lti_problem(16100, form=form, order=3, batch=2, length=30000, dtype="f64", a0=1.7, angles="spread")
    check(p)


def test_config4_full_three_phase():
    c = inputs.CONFIGS["c4"]
    p = inputs.lti_problem(1004, form=c["form"], order=c["order"], batch=1, length=c["length"], dtype="f32",
                           angles="spread")
    check(p)


def test_config5_shard_three_phase():
    p = inputs.lti_problem(1005, form="tdf", order=8, batch=256, length=1 << 16, dtype="f32", angles="spread")
    check(p)


def test_config2_three_phase():
    c = inputs.CONFIGS["c2"]
    p = inputs.lti_problem(1002, form=c["form"], order=c["order"], batch=c["batch"], length=c["length"],
                           dtype=c["dtype"], angles=c["angles"])
    check(p)


@pytest.mark.parametrize("fwd,bwd", [(P1, P3), (P3, P1)])
def test_mixed_schedules(fwd, bwd):
    """Forward and backward schedules are independent (same tape / workspace layout)."""
    p = inputs.lti_problem(17000, form="df", order=5, batch=4, length=70001, dtype="f32", angles="spread")
    check(p, flags=fwd, flags_bwd=bwd)


def test_schedules_agree():
    """Single pass and three-phase differ only in the fp64 rounding of the carries."""
    p = inputs.lti_problem(17100, form="tdf", order=6, batch=9, length=123457, dtype="f64", angles="spread")
    g1 = run_lti_gpu(p, flags=P1)
    g3 = run_lti_gpu(p, flags=P3)
    for k in g1:
        assert nrm_err(g3[k], g1[k]) < 1e-12, k


def test_deterministic_bitwise():
    p = inputs.lti_problem(18000, form="tdf", order=6, batch=16, length=50000, dtype="f32", angles="spread")
    g1 = run_lti_gpu(p, flags=P3)
    g2 = run_lti_gpu(p, flags=P3, repeat=2)
    for k in g1:
        assert np.array_equal(g1[k], g2[k]), k


def test_null_optional_outputs():
    p = inputs.lti_problem(18100, form="df", order=3, batch=2, length=50000, dtype="f32", zi=False, gzf=False)
    g = run_lti_gpu(p, want=("y", "gx"), flags=P3)
    o = run_lti_oracle(p)
    errs, bad = compare(g, o, TOL["f32"], keys=("y", "gx"))
    assert not bad, errs


def test_unaligned_rows_scalar_path():
    p = inputs.lti_problem(18200, form="tdf", order=2, batch=4, length=40099, dtype="f32")
    check(p)


def test_cuda_graph_capture_three_phase():
    p = inputs.lti_problem(18400, form="tdf", order=4, batch=8, length=100000, dtype="f32", zi=False, gzf=False,
                           angles="spread")
    td = torch.float32
    x, b, a, gy = (torch.tensor(p[k], dtype=td, device="cuda") for k in ("x", "b", "a", "gy"))
    desc = B.make_desc(8, 100000, 4, "tdf", td, 0, flags=P3)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    tape = torch.empty(tb, dtype=torch.uint8, device="cuda")
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    y, gx = torch.empty_like(x), torch.empty_like(x)
    gb, ga = torch.empty_like(b), torch.empty_like(a)
    B.iir_workspace_init(desc, ws, wb)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            B.iir_forward(desc, b, a, x, None, y, None, tape, tb, ws, wb, s)
            B.iir_backward(desc, gy, None, b, a, x, y, None, tape, tb, gx, gb, ga, None, ws, wb, s)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    o = run_lti_oracle(p)
    for k, v in (("y", y), ("gx", gx), ("gb", gb), ("ga", ga)):
        assert nrm_err(v.double().cpu().numpy(), o[k]) < 1e-4, k
