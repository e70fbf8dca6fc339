"""Seeded synthetic input generators (shared by tests and bench.py).

This module holds NONE of the method's arithmetic (no filtering, no
gradients): it only draws random stable coefficient sets and signals with the
shapes / distributions of the paper's workloads (audio-rate
signals, M = 2 biquads, N = 2^14..2^20) and of BASELINE.json's configs.  The
recipe is stated in DESIGN.md ("Input recipe") and follows SURVEY.md §8(d):

* poles: conjugate pairs r e^{+-i theta}; r ~ U(r_lo, r_hi); angles either
  uniform in (0.02 pi, 0.98 pi) ("random") or spread, theta_j =
  pi (j + 0.5 + U(-0.3, 0.3)) / P for P pairs ("spread"); an odd order adds
  one real pole of radius U(r_lo, r_hi) and random sign.
* a = monic polynomial with those roots; b ~ N(0, 1).
* x, grad_y, grad_zf ~ N(0, 1); zi ~ 0.1 N(0, 1).
* every value is rounded to the requested dtype BEFORE either side sees it
  (so the fp64 oracle and the fp32 kernel get bit-identical inputs).
* time-varying all-pole (config 3): per 256-sample frame draw 12 spread
  pole pairs, r ~ U(0.3, 0.95); map to reflection coefficients (step-down),
  interpolate them linearly per sample, map back (step-up) to a(n).
"""
from __future__ import annotations

import numpy as np
import torch

CONFIGS = {
    # name: (form, M, B, T, dtype, coef_mode, pole recipe)
    "c1": dict(form="tdf", order=2, batch=1, length=4096, dtype="f64", coef="shared", angles="random"),
    "c2": dict(form="tdf", order=2, batch=64, length=1 << 16, dtype="f32", coef="shared", angles="random"),
    "c3": dict(form="df", order=24, batch=32, length=1 << 18, dtype="f32", coef="per_sample", angles="spread"),
    "c4": dict(form="tdf", order=4, batch=1, length=1 << 24, dtype="f32", coef="shared", angles="spread"),
    "c5": dict(form="tdf", order=8, batch=2048, length=1 << 16, dtype="f32", coef="shared", angles="spread"),
    # the bare recurrence the paper benchmarks (M = 2, N = 2^14 .. 2^20)
    "f1": dict(form="ss", order=2, batch=64, length=1 << 20, dtype="f32", coef="shared", angles="random"),
}


def np_dtype(dtype: str):
    return {"f32": np.float32, "f64": np.float64}[dtype]


def torch_dtype(dtype: str):
    return {"f32": torch.float32, "f64": torch.float64}[dtype]


def random_poles(rng: np.random.Generator, order: int, r_lo=0.5, r_hi=0.99, angles="random"):
    pairs = order // 2
    r = rng.uniform(r_lo, r_hi, size=pairs)
    if angles == "spread" and pairs > 0:
        th = np.pi * (np.arange(pairs) + 0.5 + rng.uniform(-0.3, 0.3, size=pairs)) / pairs
    else:
        th = rng.uniform(0.02 * np.pi, 0.98 * np.pi, size=pairs)
    poles = list(r * np.exp(1j * th)) + list(r * np.exp(-1j * th))
    if order % 2:
        poles.append(rng.uniform(r_lo, r_hi) * rng.choice([-1.0, 1.0]))
    return np.array(poles)


def stable_coefs(rng, order, dtype="f64", r_lo=0.5, r_hi=0.99, angles="random", a0=1.0):
    """(b, a) of one stable filter of the given order, rounded to dtype."""
    p = random_poles(rng, order, r_lo, r_hi, angles)
    a = np.real(np.poly(p)) * a0
    b = rng.standard_normal(order + 1)
    t = np_dtype(dtype)
    return b.astype(t).astype(np.float64), a.astype(t).astype(np.float64)


def rbj_peaking(f0, q, gain_db, fs=48000.0):
    """RBJ cookbook peaking EQ biquad (stress set; reported, not gated)."""
    A = 10 ** (gain_db / 40)
    w0 = 2 * np.pi * f0 / fs
    alpha = np.sin(w0) / (2 * q)
    b = np.array([1 + alpha * A, -2 * np.cos(w0), 1 - alpha * A])
    a = np.array([1 + alpha / A, -2 * np.cos(w0), 1 - alpha / A])
    return b / a[0], a / a[0]


def lti_problem(seed, form="tdf", order=2, batch=1, length=4096, dtype="f32", coef="shared",
                angles="random", zi=True, gzf=True, a0=1.0, r_hi=0.99):
    """Inputs for one LTI problem as float64 numpy arrays rounded to dtype."""
    rng = np.random.default_rng(seed)
    t = np_dtype(dtype)
    if coef == "shared":
        b, a = stable_coefs(rng, order, dtype, angles=angles, a0=a0, r_hi=r_hi)
    else:
        bs, as_ = zip(*[stable_coefs(rng, order, dtype, angles=angles, a0=a0, r_hi=r_hi)
                        for _ in range(batch)])
        b, a = np.stack(bs), np.stack(as_)
    rnd = lambda *s: rng.standard_normal(s).astype(t).astype(np.float64)
    x = rnd(batch, length)
    gy = rnd(batch, length)
    p = dict(form=form, b=b, a=a, x=x, gy=gy,
             zi=(0.1 * rnd(batch, order)).astype(t).astype(np.float64) if zi else None,
             gzf=rnd(batch, order) if gzf else None, dtype=dtype)
    return p


# ---- reflection-coefficient <-> polynomial maps (Levinson step-up/down) ----
def poly_to_reflection(a):
    """Step-down: monic a[..., 0..M] -> reflection k[..., 1..M] (float64)."""
    a = np.array(a, dtype=np.float64)
    M = a.shape[-1] - 1
    k = np.zeros(a.shape[:-1] + (M,))
    cur = a[..., 1:].copy()
    for m in range(M, 0, -1):
        km = cur[..., m - 1].copy()
        k[..., m - 1] = km
        if m > 1:
            rev = cur[..., :m - 1][..., ::-1]
            cur = (cur[..., :m - 1] - km[..., None] * rev) / (1 - km[..., None] ** 2)
    return k


def reflection_to_poly_torch(k):
    """Step-up on a torch tensor k[..., M] -> a[..., 1..M] (no leading 1)."""
    M = k.shape[-1]
    a = k[..., :1].clone()
    for m in range(2, M + 1):
        km = k[..., m - 1:m]
        a = torch.cat([a + km * a.flip(-1), km], dim=-1)
    return a


def tv_allpole_problem(seed, batch=32, length=1 << 18, order=24, hop=256, dtype="f32",
                       zi=True, gzf=True, device="cpu"):
    """Config-3 inputs: a (B, T, M) per-sample all-pole coefficients."""
    rng = np.random.default_rng(seed)
    nf = (length + hop - 1) // hop + 1
    frames = np.empty((batch, nf, order + 1))
    for i in range(batch):
        for f in range(nf):
            p = random_poles(rng, order, 0.3, 0.95, angles="spread")
            frames[i, f] = np.real(np.poly(p))
    kf = torch.from_numpy(poly_to_reflection(frames)).to(device)            # (B, nf, M)
    n = torch.arange(length, device=device, dtype=torch.float64)
    f0 = torch.div(n, hop, rounding_mode="floor").long()
    w = ((n - f0 * hop) / hop)[None, :, None]
    k = kf[:, f0] * (1 - w) + kf[:, f0 + 1] * w                              # (B, T, M)
    a = reflection_to_poly_torch(k)
    td = torch_dtype(dtype)
    a = a.to(td).to(torch.float64)
    g = torch.Generator(device="cpu").manual_seed(seed + 1)
    rnd = lambda *s: torch.randn(*s, generator=g, dtype=torch.float64).to(td).to(torch.float64).to(device)
    return dict(a=a, x=rnd(batch, length), gy=rnd(batch, length),
                zi=(0.1 * rnd(batch, order)).to(td).to(torch.float64) if zi else None,
                gzf=rnd(batch, order) if gzf else None, dtype=dtype)


def tv_df_problem(seed, batch=4, length=1 << 14, order=8, hop=256, dtype="f32", zi=True, gzf=True, device="cpu"):
    """General time-varying DF inputs: the config-3 all-pole recipe
    for a(n) plus a per-sample numerator b(n) (B, T, M+1): per frame b ~ N(0, 1/(M+1)),
    linearly interpolated per sample (the frame-interpolated synthesis shape)."""
    p = tv_allpole_problem(seed, batch=batch, length=length, order=order, hop=hop, dtype=dtype, zi=zi, gzf=gzf,
                           device=device)
    rng = np.random.default_rng(seed + 7)
    nf = (length + hop - 1) // hop + 1
    bf = torch.from_numpy(rng.standard_normal((batch, nf, order + 1)) / np.sqrt(order + 1)).to(device)
    n = torch.arange(length, dtype=torch.float64, device=device)
    f0 = torch.div(n, hop, rounding_mode="floor").long()
    w = ((n - f0 * hop) / hop)[None, :, None]
    b = bf[:, f0] * (1 - w) + bf[:, f0 + 1] * w
    p["b"] = b.to(torch_dtype(dtype)).to(torch.float64)
    return p


def stable_matrix(rng, order, r_lo=0.5, r_hi=0.99):
    """Dense stable A (order x order): rotation-scaling blocks r R(theta) (and one
    real eigenvalue for odd orders) conjugated by a random orthogonal matrix, so
    A is normal (well-conditioned eigenvectors) with spectral radius <= r_hi."""
    A = np.zeros((order, order))
    i = 0
    while i + 1 < order:
        r = rng.uniform(r_lo, r_hi)
        th = rng.uniform(0.02 * np.pi, 0.98 * np.pi)
        A[i:i + 2, i:i + 2] = r * np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
        i += 2
    if i < order:
        A[i, i] = rng.uniform(r_lo, r_hi) * rng.choice([-1.0, 1.0])
    Q, _ = np.linalg.qr(rng.standard_normal((order, order)))
    return Q @ A @ Q.T


def rec_problem(seed, batch=2, length=4096, order=2, dtype="f32", coef="shared", v0=True, r_hi=0.99):
    """Inputs of the bare recurrence v(n+1) = A v(n) + z(n) (Listing 1), float64
    numpy rounded to dtype: A (M, M) or (B, M, M), v0 (B, M), z, gv (B, N, M)."""
    rng = np.random.default_rng(seed)
    t = np_dtype(dtype)
    r = lambda a: np.asarray(a).astype(t).astype(np.float64)
    if coef == "shared":
        A = r(stable_matrix(rng, order, r_hi=r_hi))
    else:
        A = r(np.stack([stable_matrix(rng, order, r_hi=r_hi) for _ in range(batch)]))
    z = r(rng.standard_normal((batch, length, order)))
    gv = r(rng.standard_normal((batch, length, order)))
    return dict(form="ss", A=A, z=z, gv=gv, v0=r(0.1 * rng.standard_normal((batch, order))) if v0 else None,
                dtype=dtype)
