"""Pins of the general time-varying DF oracle (orc_tv_df; SURVEY 8(f) f2,
reading R19: b(n) and monic a(n) both apply at output time n,
u(n) = x(n) - sum_i a_i(n) u(n-i), y(n) = sum_k b_k(n) u(n-k)).  Each pin is
independent of the oracle's dense state-space coding: scipy's lfilter for
constant coefficients, the pinned LTI / all-pole oracles as special cases,
torch autograd through the two difference equations written out, and central
finite differences."""
import numpy as np
import pytest
import scipy.signal
import torch

from paper_2511_14390_b200 import inputs


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    s = np.sqrt(np.mean(b ** 2))
    return np.max(np.abs(a - b)) / (s if s > 0 else 1.0)


def tvdf_problem(seed, B, N, M, r_hi=0.9):
    """Slowly varying stable a(n) (interpolated between two stable sets), b(n) ~ smooth + noise."""
    rng = np.random.default_rng(seed)
    a = np.empty((B, N, M))
    b = np.empty((B, N, M + 1))
    for i in range(B):
        b1, a1 = inputs.stable_coefs(rng, M, "f64", r_hi=r_hi, angles="spread")
        b2, a2 = inputs.stable_coefs(rng, M, "f64", r_hi=r_hi, angles="spread")
        w = np.linspace(0, 1, N)[:, None]
        a[i] = (1 - w) * a1[1:] + w * a2[1:]
        b[i] = (1 - w) * b1 + w * b2
    x = rng.standard_normal((B, N))
    zi = 0.3 * rng.standard_normal((B, M))
    gy = rng.standard_normal((B, N))
    gzf = rng.standard_normal((B, M))
    return b, a, x, zi, gy, gzf


@pytest.mark.parametrize("M", [1, 2, 5])
def test_constant_coefficients_equal_scipy_lfilter(orc, M):
    b, a, x, _, _, _ = tvdf_problem(300 + M, 2, 200, M)
    b[:] = b[:, :1, :]
    a[:] = a[:, :1, :]
    o = orc.tv_df(b, a, x)
    for i in range(2):
        ref = scipy.signal.lfilter(b[i, 0], np.r_[1.0, a[i, 0]], x[i])
        assert rel(o["y"][i], ref) < 1e-12


@pytest.mark.parametrize("M", [2, 4])
def test_constant_coefficients_equal_lti_df_oracle(orc, M):
    """With zi, grad_y, grad_zf: every output equals the (scipy / autograd pinned)
    LTI DF oracle; the per-sample coefficient gradients sum to the LTI ones."""
    b, a, x, zi, gy, gzf = tvdf_problem(310 + M, 2, 120, M)
    b[:] = b[:, :1, :]
    a[:] = a[:, :1, :]
    o = orc.tv_df(b, a, x, zi, gy, gzf)
    l = orc.lti(0, b[:, 0], np.concatenate([np.ones((2, 1)), a[:, 0]], axis=1), x, zi, gy, gzf)
    for k in ("y", "zf", "gx", "gzi"):
        assert rel(o[k], l[k]) < 1e-12, k
    assert rel(o["gb"].sum(axis=1), l["gb"]) < 1e-12
    assert rel(o["ga"].sum(axis=1), l["ga"][:, 1:]) < 1e-12


def test_unit_numerator_equals_tv_allpole(orc):
    b, a, x, zi, gy, gzf = tvdf_problem(320, 2, 150, 4)
    b[:] = 0.0
    b[:, :, 0] = 1.0
    o = orc.tv_df(b, a, x, zi, gy, gzf)
    p = orc.tv_allpole(a, x, zi, gy, gzf)
    for k in ("y", "zf", "gx", "ga", "gzi"):
        assert rel(o[k], p[k]) < 1e-12, k


def autograd_reference(b, a, x, zi, gy, gzf):
    """The definition, written out sample by sample in torch fp64."""
    t = lambda v: torch.tensor(v, dtype=torch.float64, requires_grad=True)
    bt, at, xt, zt = t(b), t(a), t(x), t(zi)
    N, M = a.shape
    u = [zt[k] for k in range(M - 1, -1, -1)]        # u(-M) .. u(-1)
    ys = []
    for n in range(N):
        un = xt[n]
        for i in range(1, M + 1):
            un = un - at[n, i - 1] * u[-i]
        u.append(un)
        yn = bt[n, 0] * un
        for k in range(1, M + 1):
            yn = yn + bt[n, k] * u[-1 - k]
        ys.append(yn)
    y = torch.stack(ys)
    zf = torch.stack([u[-k] for k in range(1, M + 1)])
    L = (y * torch.tensor(gy)).sum() + (zf * torch.tensor(gzf)).sum()
    L.backward()
    return dict(y=y.detach().numpy(), zf=zf.detach().numpy(), gx=xt.grad.numpy(), gb=bt.grad.numpy(),
                ga=at.grad.numpy(), gzi=zt.grad.numpy())


@pytest.mark.parametrize("M,N", [(1, 1), (2, 2), (3, 40), (5, 3), (4, 64)])
def test_all_outputs_equal_autograd_of_the_definition(orc, M, N):
    b, a, x, zi, gy, gzf = tvdf_problem(330 + M + N, 1, N, M)
    o = orc.tv_df(b, a, x, zi, gy, gzf)
    r = autograd_reference(b[0], a[0], x[0], zi[0], gy[0], gzf[0])
    for k in ("y", "zf", "gx", "gb", "ga", "gzi"):
        assert rel(o[k][0], r[k]) < 1e-12, k


def test_gradients_equal_central_finite_differences(orc):
    M, N = 3, 9
    b, a, x, zi, gy, gzf = tvdf_problem(340, 1, N, M)
    o = orc.tv_df(b, a, x, zi, gy, gzf)

    def loss(bb, aa, xx, zz):
        q = orc.tv_df(bb, aa, xx, zz)
        return float((q["y"] * gy).sum() + (q["zf"] * gzf).sum())

    args = [b, a, x, zi]
    grads = [o["gb"], o["ga"], o["gx"], o["gzi"]]
    rng = np.random.default_rng(3)
    for ai, (arr, g) in enumerate(zip(args, grads)):
        for _ in range(4):
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            h = 1e-6 * max(1.0, abs(arr[idx]))
            p, m = [v.copy() for v in args], [v.copy() for v in args]
            p[ai][idx] += h
            m[ai][idx] -= h
            fd = (loss(*p) - loss(*m)) / (2 * h)
            assert abs(fd - g[idx]) <= 1e-6 * max(1.0, abs(fd)), (ai, idx, fd, g[idx])
