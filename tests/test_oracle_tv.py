"""Pins of the time-varying all-pole oracle (orc_tv_allpole; reading R10/R11
of DESIGN.md, PAPER.md:178 'easily extended to parameter-varying cases')."""
import numpy as np
import pytest
import torch

from paper_2511_14390_b200 import inputs


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    s = np.sqrt(np.mean(b ** 2))
    return np.max(np.abs(a - b)) / (s if s > 0 else 1.0)


def tv_problem(seed, B, N, M, r_hi=0.9):
    rng = np.random.default_rng(seed)
    # slowly varying stable coefficients: interpolate between two stable sets
    a = np.empty((B, N, M))
    for i in range(B):
        _, a1 = inputs.stable_coefs(rng, M, "f64", r_hi=r_hi, angles="spread")
        _, a2 = inputs.stable_coefs(rng, M, "f64", r_hi=r_hi, angles="spread")
        w = np.linspace(0, 1, N)[:, None]
        a[i] = (1 - w) * a1[1:] + w * a2[1:]
    x = rng.standard_normal((B, N))
    zi = 0.3 * rng.standard_normal((B, M))
    gy = rng.standard_normal((B, N))
    gzf = rng.standard_normal((B, M))
    return a, x, zi, gy, gzf


@pytest.mark.parametrize("M", [1, 2, 4, 7])
def test_constant_coefficients_reduce_to_lti_allpole(orc, M):
    """a(n) == a for all n is the LTI DF filter b = [1, 0, ..], a = [1, a]
    (whose DF state [u(n-1)..u(n-M)] = [y(n-1)..y(n-M)])."""
    a, x, zi, gy, gzf = tv_problem(200 + M, 2, 150, M)
    a[:] = a[:, :1, :]
    o = orc.tv_allpole(a, x, zi, gy, gzf)
    for i in range(2):
        bb = np.zeros(M + 1)
        bb[0] = 1
        aa = np.concatenate([[1.0], a[i, 0]])
        l = orc.lti(0, bb, aa, x[i], zi=zi[i], gy=gy[i], gzf=gzf[i])
        assert rel(o["y"][i], l["y"]) < 1e-13
        assert np.max(np.abs(o["zf"][i] - l["zf"])) < 1e-12
        assert rel(o["gx"][i], l["gx"]) < 1e-13
        assert np.max(np.abs(o["gzi"][i] - l["gzi"])) < 1e-11
        assert rel(o["ga"][i].sum(axis=0), l["ga"][1:]) < 1e-12


def torch_tv(a, x, zi, gy, gzf):
    """y(n) = x(n) - sum_i a_i(n) y(n-i), y(-k) = zi[k-1], looped naively."""
    M = a.shape[-1]
    hist = [zi[k] for k in range(M)]
    ys = []
    for n in range(x.shape[0]):
        yn = x[n] - sum(a[n, i] * hist[i] for i in range(M))
        ys.append(yn)
        hist = [yn] + hist[:-1]
    return (torch.stack(ys) * gy).sum() + (torch.stack(hist) * gzf).sum()


@pytest.mark.parametrize("M,N", [(1, 1), (3, 2), (2, 30), (5, 41), (4, 3)])
def test_tv_backward_equals_autograd(orc, M, N):
    a, x, zi, gy, gzf = tv_problem(300 + M * N, 1, N, M)
    T = lambda v: torch.tensor(v, dtype=torch.float64, requires_grad=True)
    ta, tx, tz = T(a[0]), T(x[0]), T(zi[0])
    torch_tv(ta, tx, tz, torch.tensor(gy[0]), torch.tensor(gzf[0])).backward()
    o = orc.tv_allpole(a, x, zi, gy, gzf)
    assert rel(o["gx"][0], tx.grad.numpy()) < 1e-12
    assert rel(o["ga"][0], ta.grad.numpy()) < 1e-12
    assert rel(o["gzi"][0], tz.grad.numpy()) < 1e-12


def test_tv_backward_equals_finite_differences(orc):
    M, N = 3, 12
    a, x, zi, gy, gzf = tv_problem(400, 1, N, M)
    o = orc.tv_allpole(a, x, zi, gy, gzf)

    def L(a_, x_, z_):
        r = orc.tv_allpole(a_, x_, z_)
        return float((r["y"] * gy).sum() + (r["zf"] * gzf).sum())

    for key, th, g in (("a", a, o["ga"]), ("x", x, o["gx"]), ("zi", zi, o["gzi"])):
        flat = th.reshape(-1)
        for i in range(0, flat.size, max(1, flat.size // 10)):
            h = 1e-5 * max(1.0, abs(flat[i]))
            p, m = th.copy(), th.copy()
            p.reshape(-1)[i] += h
            m.reshape(-1)[i] -= h
            args = lambda t: (t if key == "a" else a, t if key == "x" else x, t if key == "zi" else zi)
            fd = (L(*args(p)) - L(*args(m))) / (2 * h)
            an = g.reshape(-1)[i]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (key, i, fd, an)


def test_generator_config3_is_stable_and_bounded():
    """The config-3 recipe gives max|a| ~ 3 and a bounded response."""
    p = inputs.tv_allpole_problem(7, batch=2, length=2048, order=24)
    a = p["a"].numpy()
    assert a.shape == (2, 2048, 24)
    assert 0.5 < np.abs(a).max() < 20
