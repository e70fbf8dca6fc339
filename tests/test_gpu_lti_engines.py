"""Both LTI engines for fp32 TDF-II against the fp64 oracle: the round-2 engine (lti2.cuh,
IIR_FLAG_ENGINE_V2: persistent warp tiles, TMEM parking, fp32 carries, fused backward) and
the round-1 engine (lti.cuh, IIR_FLAG_LEGACY_LTI), whichever the default dispatch picks for
a shape.  Gate: 1e-4 of max|gpu - oracle| / rms(oracle) per output tensor."""
import numpy as np
import pytest

from paper_2511_14390_b200 import _binding as B
from paper_2511_14390_b200 import inputs

from gpu_util import TOL, compare, run_lti_gpu, run_lti_oracle

pytestmark = pytest.mark.gpu

ENGINES = {"v2": B.IIR_FLAG_ENGINE_V2, "v1": B.IIR_FLAG_LEGACY_LTI}
TS2 = 2048                                            # round-2 tile: 32 lanes x 64 samples


def check(p, engine, seqs=None):
    g = run_lti_gpu(p, flags=ENGINES[engine])
    o = run_lti_oracle(p, seqs)
    errs, bad = compare(g, o, TOL[p["dtype"]], seqs=seqs)
    assert not bad, f"{engine}: errors {errs} exceed {TOL[p['dtype']]}"
    return errs


@pytest.mark.parametrize("engine", ["v2", "v1"])
@pytest.mark.parametrize("cfg", ["c2", "c4", "c5"])
def test_baseline_configs(engine, cfg):
    c = dict(inputs.CONFIGS[cfg])
    if cfg == "c5":
        c["batch"] = 256                              # one GPU's shard
    p = inputs.lti_problem(1000 + int(cfg[1]), form="tdf", order=c["order"], batch=c["batch"], length=c["length"],
                           dtype="f32", angles=c["angles"])
    check(p, engine)


@pytest.mark.parametrize("engine", ["v2", "v1"])
@pytest.mark.parametrize("M", [1, 2, 3, 4, 5, 6, 7, 8])
def test_orders(engine, M):
    p = inputs.lti_problem(12000 + M, form="tdf", order=M, batch=3, length=3 * TS2 + 77, dtype="f32",
                           angles="spread")
    check(p, engine)


@pytest.mark.parametrize("engine", ["v2", "v1"])
@pytest.mark.parametrize("T", [1, 2, 3, 5, 8, 63, 64, 65, 2047, 2048, 2049, 4095, 4097, 6143, 10007])
def test_edge_lengths(engine, T):
    p = inputs.lti_problem(13000 + T, form="tdf", order=3, batch=2, length=T, dtype="f32")
    check(p, engine)


@pytest.mark.parametrize("engine", ["v2", "v1"])
@pytest.mark.parametrize("zi,gzf", [(False, False), (True, False), (False, True)])
def test_initial_condition_paths(engine, zi, gzf):
    p = inputs.lti_problem(14000, form="tdf", order=8, batch=5, length=20000, dtype="f32", zi=zi, gzf=gzf,
                           angles="spread")
    check(p, engine)


@pytest.mark.parametrize("engine", ["v2", "v1"])
@pytest.mark.parametrize("M", [2, 8])
def test_per_sequence_coefficients(engine, M):
    p = inputs.lti_problem(15000 + M, form="tdf", order=M, batch=7, length=5 * TS2 + 5, dtype="f32",
                           coef="per_seq", angles="spread")
    check(p, engine)


@pytest.mark.parametrize("engine", ["v2", "v1"])
@pytest.mark.parametrize("a0", [1.7, -0.6])
def test_unnormalised_a0(engine, a0):
    p = inputs.lti_problem(16000, form="tdf", order=6, batch=2, length=9000, dtype="f32", a0=a0, angles="spread",
                           r_hi=0.9)
    check(p, engine)


@pytest.mark.parametrize("engine", ["v2"])
@pytest.mark.parametrize("ntiles", [31, 32, 33, 63, 64, 65, 1023, 1024, 1025, 1057])
def test_v2_lookback_levels(engine, ntiles):
    """Round-2 tile counts around the base-32 look-back levels (closing tiles publish
    block aggregates at aggregate time) on one sequence."""
    p = inputs.lti_problem(17000 + ntiles, form="tdf", order=4, batch=1, length=ntiles * TS2 - 3, dtype="f32",
                           angles="spread")
    check(p, engine)


@pytest.mark.parametrize("engine", ["v2"])
def test_v2_bitwise_deterministic_per_seq(engine):
    p = inputs.lti_problem(18000, form="tdf", order=7, batch=9, length=7 * TS2 + 11, dtype="f32", coef="per_seq",
                           angles="spread")
    g1 = run_lti_gpu(p, flags=ENGINES[engine])
    g2 = run_lti_gpu(p, flags=ENGINES[engine])
    for k in g1:
        assert np.array_equal(g1[k], g2[k]), k


@pytest.mark.parametrize("M,T", [(4, 3 * TS2 + 77), (8, 9 * TS2), (6, 1000), (8, 1 << 16)])
def test_v2_grad_y_early(M, T):
    """IIR_FLAG_GRAD_Y_EARLY (grad_y written before the forward): the round-2 backward loads dy,
    aggregates and publishes its first tile before waiting for the forward; same results."""
    p = inputs.lti_problem(19000 + M, form="tdf", order=M, batch=5, length=T, dtype="f32", angles="spread")
    g = run_lti_gpu(p, flags=B.IIR_FLAG_ENGINE_V2 | B.IIR_FLAG_GRAD_Y_EARLY)
    o = run_lti_oracle(p)
    errs, bad = compare(g, o, TOL["f32"])
    assert not bad, f"errors {errs}"
    g2 = run_lti_gpu(p, flags=B.IIR_FLAG_ENGINE_V2)
    for k in g:
        if g[k] is not None:
            assert np.array_equal(g[k], g2[k]), k                # bitwise the same as without the flag
