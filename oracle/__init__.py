"""fp64 CPU oracle for arXiv 2511.14390 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product path
(``paper_2511_14390_b200``) never imports it and shares no code with it.

The arithmetic lives in ``iir_oracle.c`` (plain C, fp64, dense state-space
matrices, sample by sample; every step cites PAPER.md).  This module only
compiles that file with gcc, loads it with ctypes and loops over the batch.

Functions
---------
lti(form, b, a, x, zi=None, gy=None, gzf=None, threads=None)
    Batched LTI DF-II (form=0) / TDF-II (form=1) forward + closed-form
    backward.  ``b``, ``a``: (M+1,) SHARED or (B, M+1) PER_SEQ.  SHARED
    gradients are summed over the batch (sum over sequences of the
    per-sequence gradients).
tv_allpole(a, x, zi=None, gy=None, gzf=None)
    Time-varying all-pole DF, a: (B, N, M).
recurrence(A, v0, z, gv=None)
    Bare Listing-1 recurrence v(n+1) = A v(n) + z(n) and its VJP.

Pinned by tests/test_oracle_*.py against scipy.signal.lfilter, closed-form
impulse / frequency responses, finite differences, torch autograd through a
naive loop, and the paper's structural identities.  Parity status of each
function is recorded in DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "iir_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile iir_oracle.c -> liboracle.so (gcc -O2, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.orc_lti.restype = ctypes.c_int
            lib.orc_lti.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_long] + [_dp] * 12
            lib.orc_tv_allpole.restype = ctypes.c_int
            lib.orc_tv_allpole.argtypes = [ctypes.c_int, ctypes.c_long] + [_dp] * 10
            lib.orc_tv_df.restype = ctypes.c_int
            lib.orc_tv_df.argtypes = [ctypes.c_int, ctypes.c_long] + [_dp] * 12
            lib.orc_tv_tdf.restype = ctypes.c_int
            lib.orc_tv_tdf.argtypes = [ctypes.c_int, ctypes.c_long] + [_dp] * 12
            lib.orc_recurrence.restype = ctypes.c_int
            lib.orc_recurrence.argtypes = [ctypes.c_int, ctypes.c_long] + [_dp] * 8
            _lib = lib
    return _lib


def _p(arr):
    if arr is None:
        return None
    return arr.ctypes.data_as(_dp)


def _f64(arr):
    if arr is None:
        return None
    return np.ascontiguousarray(np.asarray(arr, dtype=np.float64))


def _nthreads(threads, n):
    if threads is None:
        threads = os.cpu_count() or 1
    return max(1, min(int(threads), n))


def lti(form, b, a, x, zi=None, gy=None, gzf=None, threads=None):
    """Batched oracle; returns dict y, zf, gx, gb, ga, gzi (numpy fp64)."""
    lib = _load()
    x = _f64(x)
    squeeze = x.ndim == 1
    if squeeze:
        x = x[None]
    B, N = x.shape
    b = _f64(b)
    a = _f64(a)
    shared = b.ndim == 1
    M = b.shape[-1] - 1
    zi = None if zi is None else _f64(zi).reshape(B, M)
    gy = None if gy is None else _f64(gy).reshape(B, N)
    gzf = None if gzf is None else _f64(gzf).reshape(B, M)
    out = dict(
        y=np.empty((B, N)), zf=np.empty((B, M)), gx=np.empty((B, N)),
        gb=np.empty((B, M + 1)), ga=np.empty((B, M + 1)), gzi=np.empty((B, M)),
    )

    def one(i):
        bi = b if shared else b[i]
        ai = a if shared else a[i]
        rc = lib.orc_lti(
            int(form), M, N, _p(bi), _p(ai), _p(x[i]),
            _p(None if zi is None else zi[i]), _p(None if gy is None else gy[i]),
            _p(None if gzf is None else gzf[i]),
            _p(out["y"][i]), _p(out["zf"][i]), _p(out["gx"][i]),
            _p(out["gb"][i]), _p(out["ga"][i]), _p(out["gzi"][i]))
        if rc != 0:
            raise ValueError(f"orc_lti failed rc={rc}")

    nt = _nthreads(threads, B)
    if nt == 1:
        for i in range(B):
            one(i)
    else:
        with ThreadPoolExecutor(nt) as ex:
            list(ex.map(one, range(B)))
    if shared:
        out["gb"] = out["gb"].sum(axis=0)
        out["ga"] = out["ga"].sum(axis=0)
    if squeeze:
        for k in ("y", "zf", "gx", "gzi"):
            out[k] = out[k][0]
        if not shared:
            out["gb"], out["ga"] = out["gb"][0], out["ga"][0]
    return out


def tv_allpole(a, x, zi=None, gy=None, gzf=None, threads=None):
    """Batched time-varying all-pole oracle; a: (B, N, M)."""
    lib = _load()
    x = _f64(x)
    B, N = x.shape
    a = _f64(a).reshape(B, N, -1)
    M = a.shape[-1]
    zi = None if zi is None else _f64(zi).reshape(B, M)
    gy = None if gy is None else _f64(gy).reshape(B, N)
    gzf = None if gzf is None else _f64(gzf).reshape(B, M)
    out = dict(y=np.empty((B, N)), zf=np.empty((B, M)), gx=np.empty((B, N)),
               ga=np.empty((B, N, M)), gzi=np.empty((B, M)))

    def one(i):
        rc = lib.orc_tv_allpole(
            M, N, _p(a[i]), _p(x[i]), _p(None if zi is None else zi[i]),
            _p(None if gy is None else gy[i]), _p(None if gzf is None else gzf[i]),
            _p(out["y"][i]), _p(out["zf"][i]), _p(out["gx"][i]), _p(out["ga"][i]),
            _p(out["gzi"][i]))
        if rc != 0:
            raise ValueError(f"orc_tv_allpole failed rc={rc}")

    nt = _nthreads(threads, B)
    if nt == 1:
        for i in range(B):
            one(i)
    else:
        with ThreadPoolExecutor(nt) as ex:
            list(ex.map(one, range(B)))
    return out


def tv_df(b, a, x, zi=None, gy=None, gzf=None, threads=None):
    """Batched general time-varying DF oracle; b: (B, N, M+1), a: (B, N, M) monic."""
    lib = _load()
    x = _f64(x)
    B, N = x.shape
    a = _f64(a).reshape(B, N, -1)
    M = a.shape[-1]
    b = _f64(b).reshape(B, N, M + 1)
    zi = None if zi is None else _f64(zi).reshape(B, M)
    gy = None if gy is None else _f64(gy).reshape(B, N)
    gzf = None if gzf is None else _f64(gzf).reshape(B, M)
    out = dict(y=np.empty((B, N)), zf=np.empty((B, M)), gx=np.empty((B, N)),
               gb=np.empty((B, N, M + 1)), ga=np.empty((B, N, M)), gzi=np.empty((B, M)))

    def one(i):
        rc = lib.orc_tv_df(
            M, N, _p(b[i]), _p(a[i]), _p(x[i]), _p(None if zi is None else zi[i]),
            _p(None if gy is None else gy[i]), _p(None if gzf is None else gzf[i]),
            _p(out["y"][i]), _p(out["zf"][i]), _p(out["gx"][i]), _p(out["gb"][i]), _p(out["ga"][i]),
            _p(out["gzi"][i]))
        if rc != 0:
            raise ValueError(f"orc_tv_df failed rc={rc}")

    nt = _nthreads(threads, B)
    if nt == 1:
        for i in range(B):
            one(i)
    else:
        with ThreadPoolExecutor(nt) as ex:
            list(ex.map(one, range(B)))
    return out


def tv_tdf(b, a, x, zi=None, gy=None, gzf=None, threads=None):
    """Batched general time-varying TDF oracle (reading R20); b: (B, N, M+1), a: (B, N, M) monic."""
    lib = _load()
    x = _f64(x)
    B, N = x.shape
    a = _f64(a).reshape(B, N, -1)
    M = a.shape[-1]
    b = _f64(b).reshape(B, N, M + 1)
    zi = None if zi is None else _f64(zi).reshape(B, M)
    gy = None if gy is None else _f64(gy).reshape(B, N)
    gzf = None if gzf is None else _f64(gzf).reshape(B, M)
    out = dict(y=np.empty((B, N)), zf=np.empty((B, M)), gx=np.empty((B, N)),
               gb=np.empty((B, N, M + 1)), ga=np.empty((B, N, M)), gzi=np.empty((B, M)))

    def one(i):
        rc = lib.orc_tv_tdf(
            M, N, _p(b[i]), _p(a[i]), _p(x[i]), _p(None if zi is None else zi[i]),
            _p(None if gy is None else gy[i]), _p(None if gzf is None else gzf[i]),
            _p(out["y"][i]), _p(out["zf"][i]), _p(out["gx"][i]), _p(out["gb"][i]), _p(out["ga"][i]),
            _p(out["gzi"][i]))
        if rc != 0:
            raise ValueError(f"orc_tv_tdf failed rc={rc}")

    nt = _nthreads(threads, B)
    if nt == 1:
        for i in range(B):
            one(i)
    else:
        with ThreadPoolExecutor(nt) as ex:
            list(ex.map(one, range(B)))
    return out


def recurrence(A, v0, z, gv=None):
    """Listing-1 bare recurrence (single sequence): returns v(1..N), gz, gv0, gA."""
    lib = _load()
    A = _f64(A)
    M = A.shape[0]
    z = _f64(z).reshape(-1, M)
    N = z.shape[0]
    v0 = _f64(v0)
    gv = None if gv is None else _f64(gv).reshape(N, M)
    v = np.empty((N, M))
    gz = np.empty((N, M))
    gv0 = np.empty(M)
    gA = np.empty((M, M))
    rc = lib.orc_recurrence(M, N, _p(A), _p(v0), _p(z), _p(gv), _p(v), _p(gz), _p(gv0), _p(gA))
    if rc != 0:
        raise ValueError(f"orc_recurrence failed rc={rc}")
    return dict(v=v, gz=gz, gv0=gv0, gA=gA)
