"""Pins of the Diag-EXT oracle (oracle/diag.py)
against things other than itself: the dense Listing-1 oracle (itself pinned to torch autograd
of Listing 1's loop and to A^n v0, tests/test_oracle_lti.py), closed forms of the scalar and
rotation recurrences, and the eigen-basis invariants.  CPU only."""
import numpy as np
import pytest

import oracle
from oracle.diag import diag_condition, diag_recurrence


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    s = np.sqrt(np.mean(b ** 2)) if b.size else 0.0
    return np.max(np.abs(a - b)) / (s if s > 0 else 1.0)


def rand_problem(rng, M, N, kind):
    if kind == "complex":                              # a complex-conjugate pole pair (M = 2) or mixed
        th = rng.uniform(0.1, 3.0)
        r = rng.uniform(0.5, 0.99)
        R = np.array([[r * np.cos(th), -r * np.sin(th)], [r * np.sin(th), r * np.cos(th)]])
        if M == 2:
            A = R
        else:
            A = np.zeros((M, M)); A[:2, :2] = R
            for i in range(2, M): A[i, i] = rng.uniform(-0.9, 0.9)
        P = rng.standard_normal((M, M)) + 2 * np.eye(M)
        A = P @ A @ np.linalg.inv(P)
    else:                                              # distinct real poles
        D = np.diag(rng.uniform(-0.95, 0.95, M))
        P = rng.standard_normal((M, M)) + 2 * np.eye(M)
        A = P @ D @ np.linalg.inv(P)
    return A, rng.standard_normal(M), rng.standard_normal((N, M)), rng.standard_normal((N, M))


@pytest.mark.parametrize("M", [1, 2, 3, 4])
@pytest.mark.parametrize("kind", ["complex", "real"])
@pytest.mark.parametrize("N", [1, 7, 300])
def test_diag_equals_dense_oracle(M, kind, N):
    """Same outputs and VJP as the dense recurrence for diagonalisable A (to kappa(V) x eps)."""
    if M == 1 and kind == "complex":
        pytest.skip("a real 1x1 A has a real pole")
    rng = np.random.default_rng(100 * M + N + (kind == "real"))
    A, v0, z, gv = rand_problem(rng, M, N, kind)
    d = diag_recurrence(A, v0, z, gv)
    o = oracle.recurrence(A, v0, z, gv)
    tol = 1e-12 * max(1.0, diag_condition(A))
    for k in ("v", "gz", "gv0", "gA"):
        assert rel(d[k], o[k]) < tol, (k, rel(d[k], o[k]))


def test_scalar_closed_form():
    """M = 1: v(n) = a^n v0 + sum_k a^(n-1-k) z(k)."""
    a, v0 = 0.9, 0.7
    z = np.linspace(-1, 1, 40)[:, None]
    d = diag_recurrence(np.array([[a]]), np.array([v0]), z)
    ref = [a ** (n + 1) * v0 + sum(a ** (n - k) * z[k, 0] for k in range(n + 1)) for n in range(40)]
    assert rel(d["v"][:, 0], ref) < 1e-13


def test_rotation_closed_form():
    """A = r R(theta): the free response is a damped rotation, v(n) = r^n R(n theta) v0."""
    r, th = 0.97, 0.3
    A = r * np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    v0 = np.array([1.0, -0.5])
    d = diag_recurrence(A, v0, np.zeros((50, 2)))
    for n in range(50):
        c, s = np.cos((n + 1) * th), np.sin((n + 1) * th)
        assert np.allclose(d["v"][n], r ** (n + 1) * np.array([[c, -s], [s, c]]) @ v0, atol=1e-13)


def test_gradients_are_linear_in_gv_and_sum_over_outputs():
    """The VJP is linear in gv, and gA / gv0 of a single unit gradient at n = 0 are closed forms:
    gv = e_i at n = 0 only -> g(0) = e_i -> gA = e_i v0^T, gv0 = A^T e_i."""
    rng = np.random.default_rng(5)
    A, v0, z, _ = rand_problem(rng, 2, 10, "complex")
    gv = np.zeros((10, 2)); gv[0, 1] = 1.0
    d = diag_recurrence(A, v0, z, gv)
    assert np.allclose(d["gA"], np.outer([0, 1], v0), atol=1e-12)
    assert np.allclose(d["gv0"], A.T @ [0, 1], atol=1e-12)
    g1 = rng.standard_normal((10, 2)); g2 = rng.standard_normal((10, 2))
    s = diag_recurrence(A, v0, z, g1 + 2 * g2)
    a1, a2 = diag_recurrence(A, v0, z, g1), diag_recurrence(A, v0, z, g2)
    assert rel(s["gA"], a1["gA"] + 2 * a2["gA"]) < 1e-12


def test_defective_matrix_has_no_usable_eigenbasis():
    """A Jordan block (repeated pole, PAPER.md:134 'only applicable when A is diagonalisable'):
    the eigenvector matrix is singular to working precision -- what the GPU path tests to fall
    back to the dense recurrence -- while a diagonalisable A with distinct poles is well conditioned."""
    J = np.array([[0.9, 1.0], [0.0, 0.9]])
    assert diag_condition(J) > 1e12
    assert diag_condition(np.array([[0.9, 0.0], [0.3, -0.5]])) < 10
