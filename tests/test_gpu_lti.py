"""GPU parity of the LTI path (iir_forward / iir_backward through the C ABI)
against the fp64 oracle on the same dtype-rounded inputs.  Gate (north star):
fp32 within 1e-4, fp64 within 1e-10 of max|gpu - oracle| / rms(oracle), per
output tensor (y, zf, grad_x, grad_b, grad_a, grad_zi)."""
import numpy as np
import pytest
import torch

from paper_2511_14390_b200 import _binding as B
from paper_2511_14390_b200 import inputs

from gpu_util import TOL, compare, run_lti_gpu, run_lti_oracle

pytestmark = pytest.mark.gpu

TS = {"f32": 4096, "f64": 2048}     # samples per tile (NT * L) for M < 4


def tile(dtype, M):
    """Samples per tile: orders from 4 up use chunks twice as long (common.cuh Chunk)."""
    return TS[dtype] * (2 if M >= 4 else 1)


def check(p, tol=None, seqs=None, **kw):
    tol = TOL[p["dtype"]] if tol is None else tol
    g = run_lti_gpu(p, **kw)
    o = run_lti_oracle(p, seqs)
    errs, bad = compare(g, o, tol, seqs=seqs)
    assert not bad, f"errors {errs} exceed {tol}"
    return errs


# ---- BASELINE.json configs -------------------------------------------------
def test_config1_tdf_biquad_fp64():
    p = inputs.lti_problem(1001, **{k: v for k, v in inputs.CONFIGS["c1"].items() if k != "coef"})
    check(p)


def test_config2_tdf_biquad_fp32_full():
    c = inputs.CONFIGS["c2"]
    p = inputs.lti_problem(1002, form=c["form"], order=c["order"], batch=c["batch"], length=c["length"],
                           dtype=c["dtype"], angles=c["angles"])
    check(p)


def test_config4_long_sequence_fp32():
    c = inputs.CONFIGS["c4"]
    p = inputs.lti_problem(1004, form=c["form"], order=c["order"], batch=1, length=c["length"],
                           dtype="f32", angles="spread")
    check(p)


def test_config5_shard_order8_fp32():
    """One GPU's shard of config 5 (256 of the 2048 sequences), full gradients."""
    p = inputs.lti_problem(1005, form="tdf", order=8, batch=256, length=1 << 16, dtype="f32", angles="spread")
    check(p)


# ---- sweeps ------------------------------------------------------------------
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("M", [1, 2, 3, 4, 5, 6, 7, 8])
def test_orders_forms_dtypes(dtype, form, M):
    p = inputs.lti_problem(2000 + M, form=form, order=M, batch=3, length=3 * tile(dtype, M) + 77, dtype=dtype,
                           angles="spread")
    check(p)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("T", [1, 2, 3, 5, 8, 31, 32, 33, 127, 4095, 4096, 4097, 2047, 2048, 2049, 8191, 10007])
def test_edge_lengths(dtype, form, T):
    p = inputs.lti_problem(3000 + T, form=form, order=3, batch=2, length=T, dtype=dtype)
    check(p)


@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("zi,gzf", [(False, False), (True, False), (False, True)])
def test_initial_condition_paths(form, zi, gzf):
    p = inputs.lti_problem(4000, form=form, order=4, batch=5, length=20000, dtype="f32", zi=zi, gzf=gzf,
                           angles="spread")
    check(p)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("form", ["tdf", "df"])
def test_per_sequence_coefficients(dtype, form):
    p = inputs.lti_problem(5000, form=form, order=4, batch=7, length=2 * TS[dtype] + 5, dtype=dtype,
                           coef="per_seq", angles="spread")
    check(p)


@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("a0", [1.7, -0.6])
def test_unnormalised_a0(form, a0):
    p = inputs.lti_problem(6000, form=form, order=3, batch=2, length=9000, dtype="f64", a0=a0, angles="spread")
    check(p)
    p = inputs.lti_problem(6001, form=form, order=3, batch=2, length=9000, dtype="f32", a0=a0, angles="spread",
                           r_hi=0.9)
    check(p)


@pytest.mark.parametrize("ntiles", [31, 32, 33, 1023, 1024, 1025])
def test_hierarchical_carry_levels(ntiles):
    """Tile counts around the base-32 level boundaries of the grid carry."""
    p = inputs.lti_problem(7100 + ntiles, form="tdf", order=2, batch=1, length=ntiles * 4096 - 5, dtype="f32",
                           angles="spread")
    check(p)


def test_workspace_reuse_without_memset():
    """IIR_FLAG_WS_READY: the workspace is cleared once; every call restores it."""
    p = inputs.lti_problem(7200, form="df", order=3, batch=5, length=70000, dtype="f32", angles="spread")
    td = torch.float32
    dev = lambda a: torch.tensor(a, dtype=td, device="cuda")
    x, b, a, zi, gy, gzf = map(dev, (p["x"], p["b"], p["a"], p["zi"], p["gy"], p["gzf"]))
    desc = B.make_desc(5, 70000, 3, "df", td, 0, flags=B.IIR_FLAG_WS_READY)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    tape = torch.empty(tb, dtype=torch.uint8, device="cuda")
    ws = torch.full((wb,), 0xAB, dtype=torch.uint8, device="cuda")
    B.iir_workspace_init(desc, ws, wb)
    o = run_lti_oracle(p)
    from gpu_util import nrm_err
    for _ in range(3):
        y, gx = torch.empty_like(x), torch.empty_like(x)
        zf, gzi = torch.empty_like(zi), torch.empty_like(zi)
        gbb, gaa = torch.empty_like(b), torch.empty_like(a)
        B.iir_forward(desc, b, a, x, zi, y, zf, tape, tb, ws, wb)
        B.iir_backward(desc, gy, gzf, b, a, x, y, zi, tape, tb, gx, gbb, gaa, gzi, ws, wb)
        torch.cuda.synchronize()
        for k, g in (("y", y), ("zf", zf), ("gx", gx), ("gb", gbb), ("ga", gaa), ("gzi", gzi)):
            assert nrm_err(g.double().cpu().numpy(), o[k]) < 1e-4, k


def test_many_tiles_one_sequence_lookback():
    """A long chain of tiles on one sequence exercises deep look-back."""
    p = inputs.lti_problem(7000, form="tdf", order=2, batch=1, length=1 << 22, dtype="f32")
    check(p)


def test_deterministic_bitwise():
    p = inputs.lti_problem(8000, form="tdf", order=6, batch=16, length=50000, dtype="f32", angles="spread")
    g1 = run_lti_gpu(p)
    g2 = run_lti_gpu(p, repeat=2)
    for k in g1:
        assert np.array_equal(g1[k], g2[k]), k


def test_null_optional_outputs():
    p = inputs.lti_problem(8100, form="df", order=3, batch=2, length=5000, dtype="f32", zi=False, gzf=False)
    g = run_lti_gpu(p, want=("y", "gx"))
    o = run_lti_oracle(p)
    errs, bad = compare(g, o, TOL["f32"], keys=("y", "gx"))
    assert not bad, errs


def test_unaligned_rows_scalar_path():
    """T not a multiple of the vector width -> scalar tile loads."""
    p = inputs.lti_problem(8200, form="tdf", order=2, batch=4, length=4099, dtype="f32")
    check(p)


def test_autograd_function_matches_oracle():
    from paper_2511_14390_b200 import lfilter
    p = inputs.lti_problem(8300, form="tdf", order=2, batch=4, length=10000, dtype="f32")
    dev = lambda a: torch.tensor(a, dtype=torch.float32, device="cuda", requires_grad=True)
    x, b, a, zi = dev(p["x"]), dev(p["b"]), dev(p["a"]), dev(p["zi"])
    y, zf = lfilter(x, b, a, zi=zi, form="tdf", return_zf=True)
    L = (y * torch.tensor(p["gy"], dtype=torch.float32, device="cuda")).sum() + \
        (zf * torch.tensor(p["gzf"], dtype=torch.float32, device="cuda")).sum()
    L.backward()
    o = run_lti_oracle(p)
    from gpu_util import nrm_err
    assert nrm_err(y.detach().cpu().numpy(), o["y"]) < 1e-4
    assert nrm_err(x.grad.cpu().numpy(), o["gx"]) < 1e-4
    assert nrm_err(b.grad.cpu().numpy(), o["gb"]) < 1e-4
    assert nrm_err(a.grad.cpu().numpy(), o["ga"]) < 1e-4
    assert nrm_err(zi.grad.cpu().numpy(), o["gzi"]) < 1e-4


def test_gradcheck_fp64_tiny():
    from paper_2511_14390_b200 import lfilter
    torch.manual_seed(0)
    x = torch.randn(2, 37, dtype=torch.float64, device="cuda", requires_grad=True)
    b = torch.tensor([0.5, -0.2, 0.1], dtype=torch.float64, device="cuda", requires_grad=True)
    a = torch.tensor([1.0, -0.6, 0.25], dtype=torch.float64, device="cuda", requires_grad=True)
    zi = torch.randn(2, 2, dtype=torch.float64, device="cuda", requires_grad=True)
    for form in ("tdf", "df"):
        f = lambda x, b, a, zi: lfilter(x, b, a, zi=zi, form=form, return_zf=True)
        assert torch.autograd.gradcheck(f, (x, b, a, zi), eps=1e-6, atol=1e-8, rtol=1e-6)


def test_cuda_graph_capture():
    """The library never syncs the host: fwd + bwd capture into a CUDA graph."""
    p = inputs.lti_problem(8400, form="tdf", order=2, batch=8, length=30000, dtype="f32")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ref = run_lti_gpu(p, stream=s)
    td = torch.float32
    x = torch.tensor(p["x"], dtype=td, device="cuda")
    b = torch.tensor(p["b"], dtype=td, device="cuda")
    a = torch.tensor(p["a"], dtype=td, device="cuda")
    gy = torch.tensor(p["gy"], dtype=td, device="cuda")
    desc = B.make_desc(8, 30000, 2, "tdf", td, 0)
    tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
    tape = torch.empty(tb, dtype=torch.uint8, device="cuda")
    ws = torch.empty(wb, dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    gx = torch.empty_like(x)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        st = torch.cuda.current_stream()
        B.iir_forward(desc, b, a, x, None, y, None, tape, tb, ws, wb, st)
        B.iir_backward(desc, gy, None, b, a, x, y, None, tape, tb, gx, None, None, None, ws, wb, st)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    o = run_lti_oracle(dict(p, zi=None, gzf=None))
    from gpu_util import nrm_err
    assert nrm_err(y.double().cpu().numpy(), o["y"]) < 1e-4
    assert nrm_err(gx.double().cpu().numpy(), o["gx"]) < 1e-4
