"""GPU parity of the Diag-EXT bare recurrence (form IIR_SS + IIR_FLAG_DIAG, SURVEY §8(f)
f3) against the dense oracle (oracle.recurrence, Listing 1)
and against the eigen-basis oracle (oracle.diag.diag_recurrence), through the C ABI.
Diag-EXT reaches the same outputs and gradients as the dense recurrence up to rounding,
so the gates are the filter gates (R13).  Sizes span several 256-sample chunks and
several 32-chunk scan blocks with a ragged tail; the defective / ill-conditioned cases
check the per-coefficient-set dense fallback."""
import numpy as np
import pytest
import torch

from oracle import diag as odiag
from paper_2511_14390_b200 import _binding as B
from paper_2511_14390_b200 import inputs

from gpu_util import TOL, nrm_err
from test_gpu_rec import check, run_gpu, run_oracle

pytestmark = pytest.mark.gpu
D = B.IIR_FLAG_DIAG


def _with_A(p, A):
    t = inputs.np_dtype(p["dtype"])
    return dict(p, A=np.asarray(A, np.float64).astype(t).astype(np.float64))


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("M", [1, 2, 3, 4])
def test_orders_dtypes(dtype, M):
    check(inputs.rec_problem(9500 + M, batch=3, length=3 * 8192 + 77, order=M, dtype=dtype), flags=D)


@pytest.mark.parametrize("N", [1, 2, 3, 255, 256, 257, 8191, 8192, 8193, 20001])
def test_lengths(N):
    check(inputs.rec_problem(9600 + N, batch=2, length=N, order=2, dtype="f32"), flags=D)


def test_per_sequence_A_and_zero_v0():
    check(inputs.rec_problem(9700, batch=5, length=9000, order=2, dtype="f32", coef="per_seq"), flags=D)
    check(inputs.rec_problem(9701, batch=2, length=5000, order=2, dtype="f64", v0=False), flags=D)
    check(inputs.rec_problem(9702, batch=3, length=4000, order=1, dtype="f32", coef="per_seq"), flags=D)


@pytest.mark.parametrize("A", [
    [[0.9, 0.3], [0.0, -0.5]],                       # real distinct eigenvalues, non-normal
    [[0.6, -0.7], [0.7, 0.6]],                       # complex pair
    [[0.8, 0.0], [0.0, 0.8]],                        # repeated, diagonalisable (A = r I)
    [[0.0, 0.5], [-0.5, 0.0]],                       # purely imaginary pair
])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_structured_matrices(A, dtype):
    p = _with_A(inputs.rec_problem(9800, batch=2, length=6000, order=2, dtype=dtype), A)
    check(p, flags=D)


@pytest.mark.parametrize("A", [
    [[0.95, 1.0], [0.0, 0.95]],                      # defective (Jordan block): kappa = inf
    [[0.9, 1.0], [0.0, 0.9 - 1e-7]],                 # near-defective: kappa ~ 1e7 > both limits
])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_dense_fallback(A, dtype):
    """Diag-EXT only applies when A is diagonalisable: the defective and
    ill-conditioned eigenbases take the dense transition and still match the oracle."""
    assert odiag.diag_condition(A) > 1e4
    p = _with_A(inputs.rec_problem(9900, batch=2, length=7000, order=2, dtype=dtype), A)
    check(p, flags=D)


def test_matches_eigenbasis_oracle():
    """Same result as the step-by-step eigen-basis oracle (oracle/diag.py steps 1-4)."""
    p = inputs.rec_problem(9950, batch=2, length=3000, order=2, dtype="f64")
    g = run_gpu(p, flags=D)
    for b in range(2):
        o = odiag.diag_recurrence(p["A"], p["v0"][b], p["z"][b], p["gv"][b])
        assert nrm_err(g["v"][b], o["v"]) <= 1e-10
        assert nrm_err(g["gz"][b], o["gz"]) <= 1e-10
        assert nrm_err(g["gv0"][b], o["gv0"]) <= 1e-10


def test_mixed_per_sequence_fallback():
    """Per-sequence A where one set is defective: only that set takes the dense path."""
    p = inputs.rec_problem(9960, batch=3, length=5000, order=2, dtype="f32", coef="per_seq")
    A = p["A"].copy()
    A[1] = [[0.95, 1.0], [0.0, 0.95]]
    check(dict(p, A=A), flags=D)


def test_same_as_dense_engine():
    """The dense engine and Diag-EXT agree with each other within the gate."""
    p = inputs.rec_problem(9970, batch=4, length=1 << 16, order=2, dtype="f32")
    g1, g2 = run_gpu(p), run_gpu(p, flags=D)
    for k in ("v", "gz", "gA", "gv0"):
        assert nrm_err(g2[k], g1[k]) <= TOL["f32"], k


def test_long_sequence():
    p = inputs.rec_problem(9980, batch=1, length=1 << 20, order=2, dtype="f32", r_hi=0.999)
    check(p, flags=D)


def test_diag_rejects_order_5():
    desc = B.make_desc(2, 100, 5, "ss", torch.float32, flags=D)
    assert B.iir_tape_bytes(desc) == 0                    # 0 = invalid descriptor (iirgrad.h)
    assert b"order must be 1..4" in B.lib().iir_last_error()


@pytest.mark.parametrize("A", [
    [[0.5, 0.2, 0.0], [-0.3, 0.6, 0.1], [0.0, 0.2, -0.7]],          # complex pair + real
    [[0.9, 0.0, 0.0], [0.1, -0.4, 0.0], [0.0, 0.3, 0.2]],           # triangular, real distinct
    [[0.0, -0.6, 0.0, 0.0], [0.6, 0.0, 0.0, 0.0], [0.0, 0.0, 0.3, 0.8], [0.0, 0.0, -0.8, 0.3]],   # two pairs
    [[0.7, 0.2, 0.1, 0.0], [0.0, 0.5, 0.3, 0.1], [0.1, 0.0, -0.6, 0.2], [0.2, 0.1, 0.0, 0.4]],    # dense
])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_structured_matrices_order_3_4(A, dtype):
    """The general eigen-decomposition (characteristic polynomial, Durand-Kerner roots,
    null vectors) on structured 3x3 / 4x4 transitions."""
    M = len(A)
    p = _with_A(inputs.rec_problem(9810 + M, batch=2, length=6000, order=M, dtype=dtype), A)
    assert odiag.diag_condition(p["A"]) < 100
    check(p, flags=D)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_dense_fallback_order_4(dtype):
    """A 4x4 transition with a Jordan block (defective): the dense fallback."""
    A = [[0.9, 1.0, 0.0, 0.0], [0.0, 0.9, 0.0, 0.0], [0.0, 0.0, 0.5, 0.2], [0.0, 0.0, -0.2, 0.5]]
    p = _with_A(inputs.rec_problem(9920, batch=2, length=7000, order=4, dtype=dtype), A)
    check(p, flags=D)


def test_matches_eigenbasis_oracle_order_4():
    p = inputs.rec_problem(9955, batch=2, length=3000, order=4, dtype="f64")
    g = run_gpu(p, flags=D)
    for b in range(2):
        o = odiag.diag_recurrence(p["A"], p["v0"][b], p["z"][b], p["gv"][b])
        assert nrm_err(g["v"][b], o["v"]) <= 1e-10
        assert nrm_err(g["gz"][b], o["gz"]) <= 1e-10


def test_autograd_diag_matches_oracle():
    from paper_2511_14390_b200 import matrix_recurrence
    p = inputs.rec_problem(9990, batch=2, length=5000, order=2, dtype="f64")
    A = torch.tensor(p["A"], device="cuda", requires_grad=True)
    v0 = torch.tensor(p["v0"], device="cuda", requires_grad=True)
    z = torch.tensor(p["z"], device="cuda", requires_grad=True)
    v = matrix_recurrence(A, v0, z, diag=True)
    (v * torch.tensor(p["gv"], device="cuda")).sum().backward()
    o = run_oracle(p)
    assert nrm_err(v.detach().cpu().numpy(), o["v"]) <= 1e-10
    assert nrm_err(z.grad.cpu().numpy(), o["gz"]) <= 1e-10
    assert nrm_err(A.grad.cpu().numpy(), o["gA"]) <= 1e-10
    assert nrm_err(v0.grad.cpu().numpy(), o["gv0"]) <= 1e-10


@pytest.mark.parametrize("A", [
    [[0.0] * 3] * 3,                                                    # zero transition (triple eigenvalue 0)
    [[0.7, 0.0, 0.0], [0.0, 0.7, 0.0], [0.0, 0.0, 0.7]],               # r I: repeated, diagonalisable
    [[0.5, 1.0, 0.0], [0.0, 0.5, 1.0], [0.0, 0.0, 0.5]],               # one Jordan block of size 3
])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_degenerate_order_3(A, dtype):
    """Repeated eigenvalues at order 3 (the general eigen-decomposition's degenerate inputs):
    whichever basis the prologue settles on (eigen or dense fallback), the result is exact."""
    p = _with_A(inputs.rec_problem(9930, batch=2, length=2000, order=3, dtype=dtype), A)
    check(p, flags=D)
