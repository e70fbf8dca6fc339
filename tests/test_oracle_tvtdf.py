"""Pins of the general time-varying TDF-II oracle (orc_tv_tdf, reading
R20: the TDF realisation of PAPER.md:67-68 at every sample, written out as the scalar
TDF-II update
    y(n) = b_0(n) x(n) + v_1(n),   v_i(n+1) = v_{i+1}(n) + b_i(n) x(n) - a_i(n) y(n),
v(0) = zi, zf = v(N)).  Each pin is independent of the oracle's dense state-space coding:
scipy's lfilter for constant coefficients (the TDF-II of scipy, zi included), the pinned
LTI TDF oracle (gradients summed over time), torch autograd through the scalar update
above, central finite differences, and the structural identity of the unit-numerator
case with the pinned all-pole oracle on skewed coefficient rows, a_i(n - i)."""
import numpy as np
import pytest
import scipy.signal
import torch

from test_oracle_tvdf import rel, tvdf_problem


@pytest.mark.parametrize("M", [1, 2, 5])
def test_constant_coefficients_equal_scipy_lfilter_with_zi(orc, M):
    b, a, x, zi, _, _ = tvdf_problem(400 + M, 2, 200, M)
    b[:] = b[:, :1, :]
    a[:] = a[:, :1, :]
    o = orc.tv_tdf(b, a, x, zi)
    for i in range(2):
        ref, zf = scipy.signal.lfilter(b[i, 0], np.r_[1.0, a[i, 0]], x[i], zi=zi[i])
        assert rel(o["y"][i], ref) < 1e-12
        assert rel(o["zf"][i], zf) < 1e-12


@pytest.mark.parametrize("M", [2, 4])
def test_constant_coefficients_equal_lti_tdf_oracle(orc, M):
    """With zi, grad_y, grad_zf: every output equals the LTI TDF oracle; the per-sample
    coefficient gradients summed over time equal the LTI ones."""
    b, a, x, zi, gy, gzf = tvdf_problem(410 + M, 2, 120, M)
    b[:] = b[:, :1, :]
    a[:] = a[:, :1, :]
    o = orc.tv_tdf(b, a, x, zi, gy, gzf)
    l = orc.lti(1, b[:, 0], np.concatenate([np.ones((2, 1)), a[:, 0]], axis=1), x, zi, gy, gzf)
    for k in ("y", "zf", "gx", "gzi"):
        assert rel(o[k], l[k]) < 1e-12, k
    assert rel(o["gb"].sum(axis=1), l["gb"]) < 1e-12
    assert rel(o["ga"].sum(axis=1), l["ga"][:, 1:]) < 1e-12


def test_unit_numerator_equals_allpole_on_skewed_rows(orc):
    """b(n) = e_0, zi = 0: y(n) = x(n) - sum_i a_i(n - i) y(n - i), i.e. the all-pole
    oracle with the skewed rows a~_i(n) = a_i(n - i) (zero before n = 0); the coefficient
    gradient maps back by the same skew."""
    M, N = 4, 150
    b, a, x, _, gy, _ = tvdf_problem(420, 2, N, M)
    b[:] = 0.0
    b[:, :, 0] = 1.0
    o = orc.tv_tdf(b, a, x, None, gy, None)
    ask = np.zeros_like(a)
    for i in range(1, M + 1):
        ask[:, i:, i - 1] = a[:, :N - i, i - 1]
    p = orc.tv_allpole(ask, x, None, gy, None)
    assert rel(o["y"], p["y"]) < 1e-12
    assert rel(o["gx"], p["gx"]) < 1e-12
    ga = np.zeros_like(a)                            # grad of a_i(m) = grad of a~_i(m + i)
    for i in range(1, M + 1):
        ga[:, :N - i, i - 1] = p["ga"][:, i:, i - 1]
    assert rel(o["ga"], ga) < 1e-12


def autograd_reference(b, a, x, zi, gy, gzf):
    """The scalar TDF-II update written out sample by sample in torch fp64."""
    t = lambda v: torch.tensor(v, dtype=torch.float64, requires_grad=True)
    bt, at, xt, zt = t(b), t(a), t(x), t(zi)
    N, M = a.shape
    v = [zt[i] for i in range(M)]                    # v_1 .. v_M
    ys = []
    for n in range(N):
        yn = bt[n, 0] * xt[n] + v[0]
        ys.append(yn)
        nv = []
        for i in range(1, M + 1):
            nxt = v[i] if i < M else torch.zeros((), dtype=torch.float64)
            nv.append(nxt + bt[n, i] * xt[n] - at[n, i - 1] * yn)
        v = nv
    y = torch.stack(ys)
    zf = torch.stack(v)
    L = (y * torch.tensor(gy)).sum() + (zf * torch.tensor(gzf)).sum()
    L.backward()
    return dict(y=y.detach().numpy(), zf=zf.detach().numpy(), gx=xt.grad.numpy(), gb=bt.grad.numpy(),
                ga=at.grad.numpy(), gzi=zt.grad.numpy())


@pytest.mark.parametrize("M,N", [(1, 1), (2, 2), (3, 40), (5, 3), (4, 64)])
def test_all_outputs_equal_autograd_of_the_scalar_update(orc, M, N):
    b, a, x, zi, gy, gzf = tvdf_problem(430 + M + N, 1, N, M)
    o = orc.tv_tdf(b, a, x, zi, gy, gzf)
    r = autograd_reference(b[0], a[0], x[0], zi[0], gy[0], gzf[0])
    for k in ("y", "zf", "gx", "gb", "ga", "gzi"):
        assert rel(o[k][0], r[k]) < 1e-12, k


def test_tdf_differs_from_df_when_coefficients_vary(orc):
    """R10 / R20: with varying rows the TDF and DF realisations are different filters
    (the same with constant rows, test above)."""
    b, a, x, zi, _, _ = tvdf_problem(440, 1, 300, 3)
    assert rel(orc.tv_tdf(b, a, x)["y"], orc.tv_df(b, a, x)["y"]) > 1e-3


def test_gradients_equal_central_finite_differences(orc):
    M, N = 3, 9
    b, a, x, zi, gy, gzf = tvdf_problem(450, 1, N, M)
    o = orc.tv_tdf(b, a, x, zi, gy, gzf)

    def loss(bb, aa, xx, zz):
        q = orc.tv_tdf(bb, aa, xx, zz)
        return float((q["y"] * gy).sum() + (q["zf"] * gzf).sum())

    args = [b, a, x, zi]
    grads = [o["gb"], o["ga"], o["gx"], o["gzi"]]
    rng = np.random.default_rng(4)
    for ai, (arr, g) in enumerate(zip(args, grads)):
        for _ in range(4):
            idx = tuple(rng.integers(0, s) for s in arr.shape)
            h = 1e-6 * max(1.0, abs(arr[idx]))
            p, m = [v.copy() for v in args], [v.copy() for v in args]
            p[ai][idx] += h
            m[ai][idx] -= h
            fd = (loss(*p) - loss(*m)) / (2 * h)
            assert abs(fd - g[idx]) <= 1e-6 * max(1.0, abs(fd)), (ai, idx, fd, g[idx])
