"""World-size-2 and -3 tests of the time-sharded driver on CPU
with the gloo backend.  The per-segment compute is the fp64 oracle (test-only
injection; the product passes dist.cuda_time_ops): its forward / backward, and
the carry P^k v built from the oracle's own free response (zf after seg_len zero
samples from zi = v; grad_zi after seg_len zero cotangents from grad_zf = v).
Every rank's segment of y and grad_x, the last rank's zf, rank 0's grad_zi and
the rank-summed coefficient gradients must equal one unsharded oracle run."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2511_14390_b200 import dist as D
from paper_2511_14390_b200 import inputs


def oracle_ops(form):
    fm = 1 if form == "tdf" else 0
    n = lambda t: None if t is None else t.numpy()
    t = lambda v: torch.from_numpy(np.ascontiguousarray(v))

    def fwd(x, b, a, zi):
        o = oracle.lti(fm, b.numpy(), a.numpy(), x.numpy(), n(zi), np.zeros(tuple(x.shape)), None)
        return t(o["y"]), t(o["zf"]), None

    def bwd(gy, gzf, b, a, x, y, zi, ctx):
        o = oracle.lti(fm, b.numpy(), a.numpy(), x.numpy(), n(zi), gy.numpy(), n(gzf))
        return t(o["gx"]), t(o["gb"]), t(o["ga"]), t(o["gzi"])        # SHARED: the oracle sums the batch

    def carry(a, W, rank, seg_len, reverse, form_):
        G, Bsz, M = W.shape
        bb = np.zeros(a.shape)
        bb[..., 0] = 1.0
        zeros = np.zeros((Bsz, seg_len))
        s = np.zeros((Bsz, M))
        order = range(G - 1, rank, -1) if reverse else range(rank)
        for j in order:
            if seg_len == 0:
                adv = s
            elif reverse:     # (A_f^T)^seg_len s: the adjoint carried over seg_len zero cotangents
                adv = oracle.lti(fm, bb, a.numpy(), zeros, None, zeros, s)["gzi"]
            else:             # A_f^seg_len s: the free response over seg_len zero samples
                adv = oracle.lti(fm, bb, a.numpy(), zeros, s, zeros, None)["zf"]
            s = adv + W[j].numpy()
        return t(s)

    return D.TimeShardOps(fwd, bwd, carry)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, form, coef, T, seg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = inputs.lti_problem(91, form=form, order=3, batch=2, length=T, dtype="f64", coef=coef, angles="spread")
        s0, s1 = rank * seg, min(T, (rank + 1) * seg)
        sl = lambda k: torch.from_numpy(np.ascontiguousarray(p[k][:, s0:s1]))
        b, a = torch.from_numpy(p["b"]), torch.from_numpy(p["a"])
        r = D.time_sharded_step(oracle_ops(form), sl("x"), sl("gy"), b, a, torch.from_numpy(p["zi"]),
                                torch.from_numpy(p["gzf"]), form, seg)
        q.put((rank, {k: getattr(r, k).numpy() for k in ("y", "zf", "gx", "gzi", "gb", "ga")}))
    except Exception as e:          # surface the worker's failure instead of a queue timeout
        q.put((rank, repr(e)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,T,seg", [(2, 300, 150), (2, 301, 200), (3, 250, 100), (3, 7, 3)])
@pytest.mark.parametrize("form", ["tdf", "df"])
@pytest.mark.parametrize("coef", ["shared", "per_seq"])
def test_time_sharded_equals_unsharded(world, T, seg, form, coef):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, form, coef, T, seg, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for r, v in res.items():
        assert isinstance(v, dict), f"rank {r}: {v}"
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = inputs.lti_problem(91, form=form, order=3, batch=2, length=T, dtype="f64", coef=coef, angles="spread")
    o = oracle.lti(1 if form == "tdf" else 0, p["b"], p["a"], p["x"], p["zi"], p["gy"], p["gzf"])
    assert o["gb"].shape == ((p["b"].shape[-1],) if coef == "shared" else p["b"].shape)
    tol = lambda got, ref: np.max(np.abs(got - ref)) / max(np.sqrt(np.mean(ref ** 2)), 1e-300)
    for r in range(world):
        s0, s1 = r * seg, min(T, (r + 1) * seg)
        assert tol(res[r]["y"], o["y"][:, s0:s1]) < 1e-11, ("y", r)
        assert tol(res[r]["gx"], o["gx"][:, s0:s1]) < 1e-11, ("gx", r)
        assert tol(res[r]["gb"], o["gb"]) < 1e-11, ("gb", r)
        assert tol(res[r]["ga"], o["ga"]) < 1e-11, ("ga", r)
    assert tol(res[world - 1]["zf"], o["zf"]) < 1e-11
    assert tol(res[0]["gzi"], o["gzi"]) < 1e-11


def test_single_rank_is_plain_step():
    """world = 1 (no process group): the driver is one forward + one backward."""
    p = inputs.lti_problem(92, form="tdf", order=2, batch=1, length=50, dtype="f64")
    T = lambda k: torch.from_numpy(np.ascontiguousarray(p[k]))
    r = D.time_sharded_step(oracle_ops("tdf"), T("x"), T("gy"), T("b"), T("a"), T("zi"), T("gzf"), "tdf", 50)
    o = oracle.lti(1, p["b"], p["a"], p["x"], p["zi"], p["gy"], p["gzf"])
    assert np.allclose(r.y.numpy(), o["y"], atol=1e-13) and np.allclose(r.gzi.numpy(), o["gzi"], atol=1e-13)
