"""Diag-EXT oracle -- TEST INFRASTRUCTURE ONLY (same rules as oracle/__init__.py:
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference may use it).

The paper's second variant of the bare recurrence (Eq.4; Listing 1,
PAPER.md:296-343), written out step by step in numpy fp64 / complex128:

  PAPER.md:132-134  "decomposing A into diagonal and invertible matrices, reducing matrix
                     multiplications to element-wise multiplications ... only applicable when
                     A is diagonalisable (i.e., no repeated poles)";
  PAPER.md:145, 167 Diag-EXT, "the extra eigen-space projection".

  1. A = V diag(lam) V^-1                                 (numpy.linalg.eig)
  2. forward in the eigen-basis: w = V^-1 v,  w(n+1) = lam * w(n) + V^-1 z(n)   (element-wise),
     v(n+1) = V w(n+1)                                    (real part: A and z are real)
  3. the VJP (Listing 1: g(N-1) = gv(N-1), g(n) = gv(n) + A^T g(n+1)) in the same basis:
     A^T = V^-T diag(lam) V^T,  h = V^T g,  h(n) = V^T gv(n) + lam * h(n+1),  g = V^-T h
  4. grad_z = g,  grad_v0 = A^T g(0),  grad_A = sum_n g(n) v(n)^T  (v(0) = v0)
     (the gradient formulas themselves are Eqs.6, 9 / Listing 1's, unchanged).

A defective or nearly defective A (repeated poles) has an ill-conditioned (or singular) V:
``diag_condition`` returns kappa(V) = ||V||_2 ||V^-1||_2, the quantity the GPU path tests
to fall back to the dense recurrence.  Pinned by tests/test_oracle_diag.py against the
dense oracle (oracle.recurrence), closed forms and invariants.
"""
from __future__ import annotations

import numpy as np


def diag_condition(A):
    """kappa_2 of the eigenvector matrix of A (inf when A is defective)."""
    A = np.asarray(A, np.float64)
    lam, V = np.linalg.eig(A)
    try:
        return float(np.linalg.cond(V))
    except np.linalg.LinAlgError:
        return float("inf")


def diag_recurrence(A, v0, z, gv=None):
    """Single sequence: A (M, M), v0 (M,), z (N, M), gv (N, M) = dL/dv(1..N).
    Returns v(1..N), gz, gv0, gA computed in the eigen-basis of A (steps 1-4 above)."""
    A = np.asarray(A, np.float64)
    M = A.shape[0]
    z = np.asarray(z, np.float64).reshape(-1, M)
    N = z.shape[0]
    v0 = np.zeros(M) if v0 is None else np.asarray(v0, np.float64)
    gv = np.zeros((N, M)) if gv is None else np.asarray(gv, np.float64).reshape(N, M)
    lam, V = np.linalg.eig(A)                          # step 1
    V = V.astype(np.complex128)
    Vi = np.linalg.inv(V)
    w = Vi @ v0                                        # step 2
    v = np.empty((N, M))
    for n in range(N):
        w = lam * w + Vi @ z[n]
        v[n] = (V @ w).real
    VT, ViT = V.T, Vi.T                                # step 3
    h = np.zeros(M, np.complex128)
    g = np.empty((N, M))
    for n in range(N - 1, -1, -1):
        h = VT @ gv[n] + lam * h
        g[n] = (ViT @ h).real
    vprev = np.vstack([v0[None, :], v[:-1]])           # step 4
    gA = g.T @ vprev
    gv0 = A.T @ g[0] if N > 0 else np.zeros(M)
    return dict(v=v, gz=g.copy(), gv0=gv0, gA=gA)
