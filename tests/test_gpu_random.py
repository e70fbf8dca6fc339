"""Randomised configurations across the whole boundary (seeded, reproducible): LTI forms,
dtypes, coefficient modes, engines and flags; per-sample DF / TDF / all-pole filters; the bare
recurrence (dense and Diag-EXT).  Every output against the fp64 oracle at the filter gates
(R13).  Shapes are drawn so that tile, segment and chunk edges are crossed."""
import numpy as np
import pytest

import oracle
from paper_2511_14390_b200 import _binding as B
from paper_2511_14390_b200 import inputs

from gpu_util import TOL, compare, run_lti_gpu, run_lti_oracle

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(20261018)
LTI_CASES = []
for i in range(24):
    form = RNG.choice(["df", "tdf"])
    dtype = RNG.choice(["f32", "f64"])
    M = int(RNG.integers(1, 9))
    Bsz = int(RNG.integers(1, 6))
    T = int(RNG.choice([RNG.integers(1, 64), RNG.integers(64, 5000), RNG.integers(5000, 40000)]))
    coef = RNG.choice(["shared", "per_seq"])
    flags = int(RNG.choice([0, B.IIR_FLAG_ENGINE_V2, B.IIR_FLAG_LEGACY_LTI, B.IIR_FLAG_GRAD_Y_EARLY]))
    zi, gzf = bool(RNG.integers(0, 2)), bool(RNG.integers(0, 2))
    LTI_CASES.append((i, str(form), str(dtype), M, Bsz, T, str(coef), flags, zi, gzf))


@pytest.mark.parametrize("case", LTI_CASES, ids=[f"lti{c[0]}-{c[1]}-{c[2]}-M{c[3]}-B{c[4]}-T{c[5]}-{c[6]}-f{c[7]}"
                                                 for c in LTI_CASES])
def test_random_lti(case):
    i, form, dtype, M, Bsz, T, coef, flags, zi, gzf = case
    p = inputs.lti_problem(40000 + i, form=form, order=M, batch=Bsz, length=T, dtype=dtype, coef=coef, zi=zi,
                           gzf=gzf, angles="spread", r_hi=0.97)
    g = run_lti_gpu(p, flags=flags)
    o = run_lti_oracle(p)
    errs, bad = compare(g, o, TOL[dtype])
    assert not bad, f"{case}: {errs}"


TV_CASES = []
for i in range(12):
    kind = RNG.choice(["allpole", "df", "tdf"])
    dtype = RNG.choice(["f32", "f64"])
    M = int(RNG.integers(1, 33))
    Bsz = int(RNG.integers(1, 4))
    T = int(RNG.choice([RNG.integers(1, 40), RNG.integers(40, 3000)]))
    TV_CASES.append((i, str(kind), str(dtype), M, Bsz, T))


@pytest.mark.parametrize("case", TV_CASES, ids=[f"tv{c[0]}-{c[1]}-{c[2]}-M{c[3]}-B{c[4]}-T{c[5]}" for c in TV_CASES])
def test_random_per_sample(case):
    i, kind, dtype, M, Bsz, T = case
    if kind == "allpole":
        from test_gpu_tv import check
        p = inputs.tv_allpole_problem(41000 + i, batch=Bsz, length=T, order=M, dtype=dtype, hop=64)
        check(p, dtype)
    elif kind == "df":
        from test_gpu_tvdf import check
        check(inputs.tv_df_problem(41100 + i, batch=Bsz, length=T, order=M, dtype=dtype, hop=64), dtype)
    else:
        from test_gpu_tvtdf import check
        check(inputs.tv_df_problem(41200 + i, batch=Bsz, length=T, order=M, dtype=dtype, hop=64), dtype)


REC_CASES = []
for i in range(8):
    dtype = RNG.choice(["f32", "f64"])
    M = int(RNG.integers(1, 5))
    Bsz = int(RNG.integers(1, 4))
    T = int(RNG.choice([RNG.integers(1, 300), RNG.integers(300, 20000)]))
    coef = RNG.choice(["shared", "per_seq"])
    diag = bool(RNG.integers(0, 2))
    REC_CASES.append((i, str(dtype), M, Bsz, T, str(coef), diag))


@pytest.mark.parametrize("case", REC_CASES, ids=[f"rec{c[0]}-{c[1]}-M{c[2]}-B{c[3]}-T{c[4]}-{c[5]}-d{int(c[6])}"
                                                 for c in REC_CASES])
def test_random_recurrence(case):
    from test_gpu_rec import check
    i, dtype, M, Bsz, T, coef, diag = case
    p = inputs.rec_problem(42000 + i, batch=Bsz, length=T, order=M, dtype=dtype, coef=coef)
    check(p, flags=B.IIR_FLAG_DIAG if diag else 0)
