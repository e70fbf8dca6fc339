"""GPU parity of the time-sharded path: iir_state_carry and the
time-sharded driver with the CUDA per-segment compute (dist.cuda_time_ops).
G ranks are simulated on the one GPU by G threads exchanging through a
barrier (the driver's comm interface; NCCL on a multi-GPU box).  Gate as for
the LTI path: fp32 1e-4, fp64 1e-10 of max|gpu - oracle| / rms(oracle), against
one unsharded fp64 oracle run on the whole sequence."""
import threading

import numpy as np
import pytest
import torch

import oracle
from paper_2511_14390_b200 import _binding as B
from paper_2511_14390_b200 import dist as D
from paper_2511_14390_b200 import inputs

from gpu_util import TOL, nrm_err

pytestmark = pytest.mark.gpu


class ThreadComm:
    """all_gather / gradient sum among G threads of one process (rank-ordered sums)."""

    def __init__(self, rank, world, shared):
        self.rank, self.world, self.sh = rank, world, shared

    def _gather(self, t):
        torch.cuda.synchronize()
        self.sh["slots"][self.rank] = t.clone()
        self.sh["bar"].wait()
        out = torch.stack([s.to(t.device) for s in self.sh["slots"]])
        self.sh["bar"].wait()
        return out

    def all_gather(self, t):
        return self._gather(t)

    def sum_grads(self, gb, ga, deterministic=False):
        g = self._gather(torch.cat([gb.reshape(-1), ga.reshape(-1)]))
        s = g[0].clone()
        for k in range(1, self.world):
            s += g[k]
        n = gb.numel()
        return s[:n].view_as(gb), s[n:].view_as(ga)


def run_sharded(p, G, seg, form):
    td = torch.float32 if p["dtype"] == "f32" else torch.float64
    dev = lambda v: torch.as_tensor(np.ascontiguousarray(v), dtype=torch.float64).to(td).cuda()
    T = p["x"].shape[1]
    sh = {"bar": threading.Barrier(G), "slots": [None] * G}
    res, errs = [None] * G, []
    streams = [torch.cuda.Stream() for _ in range(G)]

    def worker(r):
        try:
            s0, s1 = r * seg, min(T, (r + 1) * seg)
            x, gy = dev(p["x"][:, s0:s1]), dev(p["gy"][:, s0:s1])
            with torch.cuda.stream(streams[r]):      # one stream per simulated rank (one GPU each on a box)
                out = D.time_sharded_step(D.cuda_time_ops(form), x, gy, dev(p["b"]), dev(p["a"]), dev(p["zi"]),
                                          dev(p["gzf"]), form, seg, comm=ThreadComm(r, G, sh))
            torch.cuda.synchronize()
            res[r] = {k: getattr(out, k).double().cpu().numpy() for k in ("y", "zf", "gx", "gzi", "gb", "ga")}
        except Exception as e:  # pragma: no cover - reported below
            errs.append(repr(e))
            sh["bar"].abort()
    th = [threading.Thread(target=worker, args=(r,)) for r in range(G)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    return res


def check(p, G, seg, form, tol=None):
    tol = TOL[p["dtype"]] if tol is None else tol
    res = run_sharded(p, G, seg, form)
    o = oracle.lti(1 if form == "tdf" else 0, p["b"], p["a"], p["x"], p["zi"], p["gy"], p["gzf"])
    assert o["gb"].shape == p["b"].shape              # SHARED: the oracle already sums over the batch
    T = p["x"].shape[1]
    errs = {}
    y = np.concatenate([res[r]["y"] for r in range(G)], axis=1)
    gx = np.concatenate([res[r]["gx"] for r in range(G)], axis=1)
    errs["y"], errs["gx"] = nrm_err(y, o["y"]), nrm_err(gx, o["gx"])
    errs["zf"], errs["gzi"] = nrm_err(res[G - 1]["zf"], o["zf"]), nrm_err(res[0]["gzi"], o["gzi"])
    errs["gb"], errs["ga"] = nrm_err(res[0]["gb"], o["gb"]), nrm_err(res[0]["ga"], o["ga"])
    for r in range(1, G):
        assert np.array_equal(res[r]["gb"], res[0]["gb"]) and np.array_equal(res[r]["ga"], res[0]["ga"])
    assert y.shape[1] == T
    assert max(errs.values()) < tol, errs
    return errs


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("M", [1, 2, 4, 8])
def test_state_carry_matches_free_response(dtype, form, M):
    """iir_state_carry against the oracle's free response: P^k v is the final
    state after k zero samples from v, (P^T)^k v the adjoint after k zero cotangents."""
    p = inputs.lti_problem(21000 + M, form=form, order=M, batch=3, length=10, dtype=dtype, angles="spread")
    td = torch.float32 if dtype == "f32" else torch.float64
    rng = np.random.default_rng(M)
    G, seg = 4, 777
    W = rng.standard_normal((G, 3, M)).astype(np.float32 if dtype == "f32" else np.float64).astype(np.float64)
    a = torch.tensor(p["a"], dtype=td, device="cuda")
    d = B.make_desc(3, seg, M, form, td, B.IIR_COEF_SHARED)
    fm = 1 if form == "tdf" else 0
    bb = np.zeros(M + 1)
    bb[0] = 1.0
    z = np.zeros((3, seg))
    for reverse in (False, True):
        for rank in range(G):
            out = torch.empty((3, M), dtype=td, device="cuda")
            B.iir_state_carry(d, a, torch.tensor(W, dtype=td, device="cuda"), G, rank, seg, reverse, out)
            s = np.zeros((3, M))
            for j in (range(G - 1, rank, -1) if reverse else range(rank)):
                adv = oracle.lti(fm, bb, p["a"], z, None, z, s)["gzi"] if reverse else \
                    oracle.lti(fm, bb, p["a"], z, s, z, None)["zf"]
                s = adv + W[j]
            torch.cuda.synchronize()
            assert nrm_err(out.double().cpu().numpy(), s) < (1e-5 if dtype == "f32" else 1e-12), (reverse, rank)


@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("G,T,seg", [(2, 20000, 10000), (3, 25001, 9000), (8, 8 * 4096, 4096), (5, 13, 3)])
def test_time_sharded_fp32(form, G, T, seg):
    p = inputs.lti_problem(22000 + G, form=form, order=3, batch=2, length=T, dtype="f32", angles="spread")
    check(p, G, seg, form)


@pytest.mark.parametrize("form", ["tdf", "df"])
def test_time_sharded_fp64_per_seq(form):
    p = inputs.lti_problem(22100, form=form, order=5, batch=3, length=30000, dtype="f64", coef="per_seq",
                           angles="spread")
    check(p, 4, 7500, form)


def test_config4_time_sharded_8_ways():
    """Config 4 (order-4 TDF, one 2^24-sample sequence, fp32) split over 8 segments."""
    c = inputs.CONFIGS["c4"]
    p = inputs.lti_problem(1004, form=c["form"], order=c["order"], batch=1, length=c["length"], dtype="f32",
                           angles="spread")
    check(p, 8, c["length"] // 8, "tdf")


def test_order8_time_sharded():
    p = inputs.lti_problem(22200, form="tdf", order=8, batch=4, length=1 << 18, dtype="f32", angles="spread")
    check(p, 4, 1 << 16, "tdf")
