"""Pins of the fp64 LTI oracle (oracle/iir_oracle.c: orc_lti) against things
other than itself: scipy's lfilter, the literal difference equations Eqs.2-3,
closed-form impulse and frequency responses, the unrolled Eq.11, torch
autograd through a naive loop, torchaudio's lfilter gradients, central finite
differences, and the paper's structural identities.  CPU only."""
import numpy as np
import pytest
import scipy.signal as ss
import torch

from paper_2511_14390_b200 import inputs

DF, TDF = 0, 1


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    s = np.sqrt(np.mean(b ** 2)) if b.size else 0.0
    return np.max(np.abs(a - b)) / (s if s > 0 else 1.0)


def problem(seed, M, N, a0=1.0, angles="random", r_hi=0.99):
    rng = np.random.default_rng(seed)
    b, a = inputs.stable_coefs(rng, M, "f64", angles=angles, a0=a0, r_hi=r_hi)
    x = rng.standard_normal(N)
    zi = 0.3 * rng.standard_normal(M)
    gy = rng.standard_normal(N)
    gzf = rng.standard_normal(M)
    return b, a, x, zi, gy, gzf


# ---------------------------------------------------------------- forward ---
@pytest.mark.parametrize("M", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("a0", [1.0, 1.7, -0.6])
def test_tdf_forward_equals_scipy_lfilter(orc, M, a0):
    """TDF-II with v(0)=zi is scipy.signal.lfilter(b, a, x, zi) (PAPER.md:58:
    TDF is 'the standard implementation' in SciPy)."""
    b, a, x, zi, _, _ = problem(10 + M, M, 300, a0=a0)
    o = orc.lti(TDF, b, a, x, zi=zi)
    y_ref, zf_ref = ss.lfilter(b, a, x, zi=zi)
    assert rel(o["y"], y_ref) < 1e-13
    assert np.max(np.abs(o["zf"] - zf_ref)) < 1e-12


def df_literal(b, a, x, u_hist):
    """Eqs.2-3 typed out literally, with past internal signal
    u(-k) = u_hist[k-1]."""
    b = np.asarray(b) / a[0]
    a = np.asarray(a) / a[0]
    M = len(a) - 1
    u = {-k: u_hist[k - 1] for k in range(1, M + 1)}
    y = np.zeros(len(x))
    for n in range(len(x)):
        u[n] = x[n] - sum(a[i] * u[n - i] for i in range(1, M + 1))
        y[n] = sum(b[i] * u[n - i] for i in range(0, M + 1))
    zf = np.array([u[len(x) - k] for k in range(1, M + 1)])
    return y, zf


@pytest.mark.parametrize("M", [1, 2, 3, 5])
@pytest.mark.parametrize("a0", [1.0, 2.5])
def test_df_forward_equals_difference_equations(orc, M, a0):
    """DF-II state space with companion(a), B=e1, C=b_k-a_k b_0, D=b_0 equals
    Eqs.2-3 (PAPER.md:66 'are equivalent to Eq.2 and Eq.3'); zi = past u."""
    b, a, x, zi, _, _ = problem(20 + M, M, 200, a0=a0)
    o = orc.lti(DF, b, a, x, zi=zi)
    y_ref, zf_ref = df_literal(b, a, x, zi)
    assert rel(o["y"], y_ref) < 1e-13
    assert np.max(np.abs(o["zf"] - zf_ref)) < 1e-12


@pytest.mark.parametrize("M", [1, 2, 4, 8])
def test_df_equals_tdf_at_zero_state(orc, M):
    """Transposition does not alter the transfer function."""
    b, a, x, _, _, _ = problem(30 + M, M, 500, angles="spread")
    assert rel(orc.lti(DF, b, a, x)["y"], orc.lti(TDF, b, a, x)["y"]) < 1e-12


@pytest.mark.parametrize("form", [DF, TDF])
def test_first_order_impulse_response_closed_form(orc, form):
    """h(n) = b0 (-a1)^n + b1 (-a1)^(n-1) for H = (b0 + b1 z^-1)/(1 + a1 z^-1)."""
    b = np.array([0.7, -1.3])
    a = np.array([1.0, -0.93])
    N = 200
    x = np.zeros(N)
    x[0] = 1.0
    h = orc.lti(form, b, a, x)["y"]
    n = np.arange(N)
    ref = b[0] * (-a[1]) ** n + np.where(n >= 1, b[1] * (-a[1]) ** np.maximum(n - 1, 0), 0.0)
    assert np.max(np.abs(h - ref)) < 1e-14


@pytest.mark.parametrize("form", [DF, TDF])
def test_allpole_biquad_impulse_closed_form(orc, form):
    """1/(1 - 2r cos(t) z^-1 + r^2 z^-2): h(n) = r^n sin((n+1)t)/sin(t)."""
    r, t = 0.97, 0.3
    b = np.array([1.0, 0.0, 0.0])
    a = np.array([1.0, -2 * r * np.cos(t), r * r])
    N = 400
    x = np.zeros(N)
    x[0] = 1.0
    h = orc.lti(form, b, a, x)["y"]
    n = np.arange(N)
    assert np.max(np.abs(h - r ** n * np.sin((n + 1) * t) / np.sin(t))) < 1e-12


@pytest.mark.parametrize("form", [DF, TDF])
@pytest.mark.parametrize("M", [2, 4])
def test_steady_state_frequency_response(orc, form, M):
    """Driving with e^{j w n} (as cos and sin runs), after the transient
    y(n) -> H(e^{jw}) e^{j w n} with H from Eq.1 on the unit circle."""
    rng = np.random.default_rng(40 + M)
    b, a = inputs.stable_coefs(rng, M, "f64", r_lo=0.3, r_hi=0.8, angles="spread")
    N = 400
    n = np.arange(N)
    for w in (0.0, 0.37, 1.9, np.pi):
        zinv = np.exp(-1j * w)
        H = np.polyval(b[::-1], zinv) / np.polyval(a[::-1], zinv)
        yc = orc.lti(form, b, a, np.cos(w * n))["y"]
        ys = orc.lti(form, b, a, np.sin(w * n))["y"]
        ref = H * np.exp(1j * w * n)
        tail = slice(300, N)  # 0.8^300 ~ 1e-29
        assert np.max(np.abs(yc[tail] - ref.real[tail])) < 1e-12
        assert np.max(np.abs(ys[tail] - ref.imag[tail])) < 1e-12
        _, Hs = ss.freqz(b, a, worN=[w])
        assert abs(H - Hs[0]) < 1e-12


@pytest.mark.parametrize("form", [DF, TDF])
def test_unrolled_matrix_power_eq11(orc, form):
    """Eq.11: v(n+1) = A^{n+1} v(0) + sum A^{n-m} z(m);
    checked through y(n) = C^T v(n) + D x(n) for N <= 8 with explicit powers."""
    M, N = 3, 8
    b, a, x, zi, _, _ = problem(50, M, N)
    A = np.zeros((M, M))
    A[0, :] = -a[1:]
    A[np.arange(1, M), np.arange(M - 1)] = 1.0
    c = b[1:] - a[1:] * b[0]
    e1 = np.eye(M)[0]
    Af, Bf, Cf = (A, e1, c) if form == DF else (A.T, c, e1)
    y = orc.lti(form, b, a, x, zi=zi)["y"]
    for nn in range(N):
        v = np.linalg.matrix_power(Af, nn) @ zi + sum(
            np.linalg.matrix_power(Af, nn - 1 - m) @ (Bf * x[m]) for m in range(nn))
        assert abs(y[nn] - (Cf @ v + b[0] * x[nn])) < 1e-12


def test_spec_worked_examples(orc):
    """Hand-derived examples (tests/golden/spec_examples.json)."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
    for ex in g["filter_forward"]:
        for form in (DF, TDF):
            y = orc.lti(form, ex["b"], ex["a"], np.array(ex["x"], float))["y"]
            assert np.array_equal(y, np.array(ex["y"], float)), ex
    for ex in g["recurrence"]:
        o = orc.recurrence(np.array(ex["A"]), np.array(ex["v0"]), np.array(ex["z"]),
                           gv=np.array(ex["gv"]) if "gv" in ex else None)
        assert np.allclose(o["v"].ravel(), ex["v"], rtol=0, atol=1e-15)
        if "gz" in ex:
            assert np.allclose(o["gz"].ravel(), ex["gz"], rtol=0, atol=1e-15)
            assert np.allclose(o["gv0"], ex["gv0"], rtol=0, atol=1e-15)
            assert np.allclose(o["gA"].ravel(), ex["gA"], rtol=0, atol=1e-15)


def test_linearity_and_superposition(orc):
    """The filter is linear in (x, zi)."""
    b, a, x, zi, _, _ = problem(60, 4, 300)
    x2 = np.random.default_rng(61).standard_normal(300)
    for form in (DF, TDF):
        f = lambda xx, z=None: orc.lti(form, b, a, xx, zi=z)["y"]
        assert rel(f(2.0 * x - 0.5 * x2), 2.0 * f(x) - 0.5 * f(x2)) < 1e-12
        assert rel(f(x, zi), f(x) + f(np.zeros_like(x), zi)) < 1e-12


# --------------------------------------------------------------- backward ---
def torch_loss(form, b, a, x, zi, gy, gzf):
    """Naive loop of the DIFFERENCE EQUATIONS (Eqs.2-3 for DF; the standard
    TDF-II recurrence for TDF), differentiated by torch autograd."""
    a0 = a[0]
    bn, an = b / a0, a / a0
    M = len(a) - 1
    ys = []
    if form == DF:
        u = [zi[k] for k in range(M)]                     # u(n-1) .. u(n-M)
        for n in range(len(x)):
            un = x[n] - sum(an[i] * u[i - 1] for i in range(1, M + 1))
            ys.append(bn[0] * un + sum(bn[i] * u[i - 1] for i in range(1, M + 1)))
            u = [un] + u[:-1]
        zf = torch.stack(u)
    else:
        s = [zi[k] for k in range(M)]
        for n in range(len(x)):
            yn = bn[0] * x[n] + s[0]
            ys.append(yn)
            s = [(s[i + 1] if i + 1 < M else 0.0) + bn[i + 1] * x[n] - an[i + 1] * yn
                 for i in range(M)]
        zf = torch.stack(s)
    y = torch.stack(ys)
    return (y * gy).sum() + (zf * gzf).sum()


@pytest.mark.parametrize("form", [DF, TDF])
@pytest.mark.parametrize("M,N,a0", [(1, 1, 1.0), (2, 2, 1.0), (3, 17, 1.4), (4, 40, -0.8), (2, 64, 1.0)])
def test_backward_equals_torch_autograd(orc, form, M, N, a0):
    b, a, x, zi, gy, gzf = problem(70 + 7 * M + N, M, N, a0=a0)
    T = lambda v: torch.tensor(v, dtype=torch.float64, requires_grad=True)
    tb, ta, tx, tzi = T(b), T(a), T(x), T(zi)
    L = torch_loss(form, tb, ta, tx, tzi, torch.tensor(gy), torch.tensor(gzf))
    L.backward()
    o = orc.lti(form, b, a, x, zi=zi, gy=gy, gzf=gzf)
    for k, ref in (("gx", tx.grad), ("gb", tb.grad), ("ga", ta.grad), ("gzi", tzi.grad)):
        assert rel(o[k], ref.numpy()) < 1e-12, k


@pytest.mark.parametrize("form", [DF, TDF])
@pytest.mark.parametrize("M,N,a0", [(1, 8, 1.0), (2, 64, 1.3), (3, 257, 1.0), (4, 8, 0.7), (2, 1, 1.0)])
def test_backward_equals_finite_differences(orc, form, M, N, a0):
    """Central differences, h = 1e-5 max(1, |theta|); the
    paper 'verified that our analytical gradients match the numerical
    gradients'."""
    b, a, x, zi, gy, gzf = problem(90 + M + N, M, N, a0=a0, r_hi=0.95)

    def L(b_, a_, x_, zi_):
        o = orc.lti(form, b_, a_, x_, zi=zi_)
        return float(np.dot(o["y"], gy) + np.dot(o["zf"], gzf))

    o = orc.lti(form, b, a, x, zi=zi, gy=gy, gzf=gzf)
    params = dict(gb=b, ga=a, gx=x, gzi=zi)
    rng = np.random.default_rng(0)
    for key, th in params.items():
        idx = range(len(th)) if len(th) <= 12 else rng.choice(len(th), 12, replace=False)
        for i in idx:
            h = 1e-5 * max(1.0, abs(th[i]))
            tp, tm = th.copy(), th.copy()
            tp[i] += h
            tm[i] -= h
            args_p = {k: (tp if k == key else v) for k, v in params.items()}
            args_m = {k: (tm if k == key else v) for k, v in params.items()}
            fd = (L(args_p["gb"], args_p["ga"], args_p["gx"], args_p["gzi"]) -
                  L(args_m["gb"], args_m["ga"], args_m["gx"], args_m["gzi"])) / (2 * h)
            an = o[key][i]
            assert abs(fd - an) <= 1e-5 * abs(an) + 1e-8 * max(1.0, abs(an)) * 10, (key, i, fd, an)


@pytest.mark.parametrize("M", [1, 2, 3, 6])
def test_backward_equals_torchaudio(orc, M):
    """torchaudio.functional.lfilter (zero initial state, clamp=False) has its
    own analytic gradient (PAPER.md:74 'implemented in TorchAudio')."""
    ta_f = pytest.importorskip("torchaudio.functional")
    b, a, x, _, gy, _ = problem(110 + M, M, 300)
    T = lambda v: torch.tensor(v, dtype=torch.float64, requires_grad=True)
    tb, ta, tx = T(b), T(a), T(x)
    y = ta_f.lfilter(tx[None], ta, tb, clamp=False)[0]
    (y * torch.tensor(gy)).sum().backward()
    for form in (DF, TDF):
        o = orc.lti(form, b, a, x, gy=gy)
        assert rel(o["y"], y.detach().numpy()) < 1e-11
        assert rel(o["gx"], tx.grad.numpy()) < 1e-10
        assert rel(o["gb"], tb.grad.numpy()) < 1e-10
        assert rel(o["ga"], ta.grad.numpy()) < 1e-10


@pytest.mark.parametrize("M", [1, 2, 5])
def test_backward_is_reverse_time_dual_filter(orc, M):
    """the backward pass of DF is a TDF filter run backwards
    in time, and vice versa: dx = flip(dual.fwd(flip(dy), zi=grad_zf)),
    grad_zi = that filter's final state."""
    b, a, x, zi, gy, gzf = problem(120 + M, M, 333)
    for form, dual in ((TDF, DF), (DF, TDF)):
        o = orc.lti(form, b, a, x, zi=zi, gy=gy, gzf=gzf)
        d = orc.lti(dual, b, a, gy[::-1].copy(), zi=gzf)
        assert rel(o["gx"], d["y"][::-1]) < 1e-13
        assert np.max(np.abs(o["gzi"] - d["zf"])) < 1e-12


def test_transpose_duality_of_gradients(orc):
    """DF and TDF share (x, dy); at zero state the gradients of
    the coefficients coincide (same transfer function => same dL/db, dL/da)."""
    b, a, x, _, gy, _ = problem(130, 4, 400)
    o1 = orc.lti(DF, b, a, x, gy=gy)
    o2 = orc.lti(TDF, b, a, x, gy=gy)
    for k in ("gx", "gb", "ga"):
        assert rel(o1[k], o2[k]) < 1e-11


def test_batched_shared_is_sum_of_sequences(orc):
    p = inputs.lti_problem(5, form="tdf", order=3, batch=5, length=100, dtype="f64")
    o = orc.lti(1, p["b"], p["a"], p["x"], p["zi"], p["gy"], p["gzf"], threads=3)
    for i in range(5):
        oi = orc.lti(1, p["b"], p["a"], p["x"][i], p["zi"][i], p["gy"][i], p["gzf"][i])
        assert np.array_equal(o["y"][i], oi["y"])
    tot = sum(orc.lti(1, p["b"], p["a"], p["x"][i], p["zi"][i], p["gy"][i], p["gzf"][i])["gb"]
              for i in range(5))
    assert rel(o["gb"], tot) < 1e-14


@pytest.mark.parametrize("M,N", [(1, 1), (2, 7), (2, 64), (3, 40), (4, 33)])
def test_recurrence_equals_autograd_of_listing1_loop(orc, M, N):
    """Bare recurrence: oracle.recurrence against torch autograd
    through the plain loop of Listing 1's forward (restated):
    v(n+1) = A v(n) + z(n), loss = sum gv * v(1..N)."""
    import torch
    from paper_2511_14390_b200 import inputs
    rng = np.random.default_rng(700 + 10 * M + N)
    A = inputs.stable_matrix(rng, M)
    v0, z, gv = rng.standard_normal(M), rng.standard_normal((N, M)), rng.standard_normal((N, M))
    At = torch.tensor(A, requires_grad=True)
    v0t = torch.tensor(v0, requires_grad=True)
    zt = torch.tensor(z, requires_grad=True)
    vn, outs = v0t, []
    for n in range(N):
        vn = At @ vn + zt[n]
        outs.append(vn)
    v = torch.stack(outs)
    (v * torch.tensor(gv)).sum().backward()
    o = orc.recurrence(A, v0, z, gv)
    np.testing.assert_allclose(o["v"], v.detach().numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(o["gz"], zt.grad.numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(o["gv0"], v0t.grad.numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(o["gA"], At.grad.numpy(), rtol=0, atol=1e-12)


def test_recurrence_closed_form_impulse():
    """v(n) = A^n v0 for z = 0 (Eq.11's unrolled form)."""
    import oracle
    from paper_2511_14390_b200 import inputs
    rng = np.random.default_rng(777)
    A = inputs.stable_matrix(rng, 3)
    v0 = rng.standard_normal(3)
    o = oracle.recurrence(A, v0, np.zeros((20, 3)))
    for n in range(1, 21):
        np.testing.assert_allclose(o["v"][n - 1], np.linalg.matrix_power(A, n) @ v0, rtol=0, atol=1e-12)
