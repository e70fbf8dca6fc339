"""World-size-2 tests of the batch-sharded driver on CPU (gloo backend).

The per-shard compute is the fp64 oracle (test-only injection; the product
passes the CUDA compute).  Checks: the shard split, that every rank's outputs
equal the corresponding slice of a single-process run, and that the
all-reduced SHARED gradients equal the full-batch gradients (both the
all_reduce and the deterministic all_gather reductions)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2511_14390_b200 import dist as D
from paper_2511_14390_b200 import inputs


def test_shard_range_covers_batch():
    for B in (1, 2, 7, 64, 2048):
        for W in (1, 2, 3, 8):
            got = [D.shard_range(B, r, W) for r in range(W)]
            assert got[0][0] == 0 and got[-1][1] == B
            for (s0, e0), (s1, e1) in zip(got, got[1:]):
                assert e0 == s1
            sizes = [e - s for s, e in got]
            assert max(sizes) - min(sizes) <= 1


def oracle_compute(x, gy, b, a, zi, gzf, form):
    import oracle
    o = oracle.lti(1 if form == "tdf" else 0, b.numpy(), a.numpy(), x.numpy(),
                   None if zi is None else zi.numpy(), gy.numpy(), None if gzf is None else gzf.numpy())
    t = lambda k: torch.from_numpy(np.ascontiguousarray(o[k]))
    return t("y"), t("zf"), t("gx"), t("gb"), t("ga"), t("gzi")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, coef, deterministic, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = inputs.lti_problem(77, form="tdf", order=3, batch=5, length=300, dtype="f64", coef=coef,
                               angles="spread")
        s0, s1 = D.shard_range(5, rank, world)
        T = lambda k: torch.from_numpy(np.ascontiguousarray(p[k][s0:s1]))
        b = torch.from_numpy(p["b"]) if coef == "shared" else T("b")
        a = torch.from_numpy(p["a"]) if coef == "shared" else T("a")
        r = D.sharded_step(oracle_compute, T("x"), T("gy"), b, a, T("zi"), T("gzf"), "tdf",
                           deterministic=deterministic)
        q.put((rank, s0, s1, {k: getattr(r, k).numpy() for k in ("y", "zf", "gx", "gzi", "gb", "ga")}))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("coef", ["shared", "per_seq"])
@pytest.mark.parametrize("deterministic", [False, True])
def test_two_rank_sharded_step_matches_single_process(orc, coef, deterministic):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, coef, deterministic, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = inputs.lti_problem(77, form="tdf", order=3, batch=5, length=300, dtype="f64", coef=coef, angles="spread")
    full = orc.lti(1, p["b"], p["a"], p["x"], p["zi"], p["gy"], p["gzf"])
    for rank, s0, s1, r in res:
        for k in ("y", "zf", "gx", "gzi"):
            np.testing.assert_allclose(r[k], full[k][s0:s1], rtol=0, atol=1e-12)
        if coef == "shared":      # all-reduced over both ranks == full-batch sum
            np.testing.assert_allclose(r["gb"], full["gb"], rtol=1e-12, atol=1e-12)
            np.testing.assert_allclose(r["ga"], full["ga"], rtol=1e-12, atol=1e-12)
        else:                     # per-sequence gradients stay local: no exchange
            np.testing.assert_allclose(r["gb"], full["gb"][s0:s1], rtol=0, atol=1e-12)
            np.testing.assert_allclose(r["ga"], full["ga"][s0:s1], rtol=0, atol=1e-12)
    if coef == "shared" and deterministic:
        assert np.array_equal(res[0][3]["gb"], res[1][3]["gb"])
