"""torch.autograd front end: ``lfilter`` and ``allpole_tv``.

Both are ``torch.autograd.Function``s whose forward calls ``iir_forward`` and
whose backward calls ``iir_backward`` of libiirgrad.so on the current CUDA
stream.  Torch only provides device memory (outputs, tape and workspace come
from its caching allocator) and streams.  CUDA tensors only: a CPU tensor is
an error, not a fallback.
"""
from __future__ import annotations

import torch

from . import _binding as B


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("paper_2511_14390_b200 runs on CUDA tensors only (no CPU fallback)")


def _check(x, named_shapes):
    """The C ABI receives raw pointers and takes the dtype from the descriptor: every
    tensor must be on x's device, have x's dtype and the exact shape of its role, or
    the kernels would read it as the wrong type / out of bounds.  Raises ValueError."""
    if x.dtype not in (torch.float32, torch.float64):
        raise ValueError(f"x must be float32 or float64, got {x.dtype}")
    for name, t, shapes in named_shapes:
        if t is None:
            continue
        if t.device != x.device:
            raise ValueError(f"{name} is on {t.device}, x on {x.device}")
        if t.dtype != x.dtype:
            raise ValueError(f"{name} has dtype {t.dtype}, x has {x.dtype}")
        if tuple(t.shape) not in [tuple(s) for s in shapes]:
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected one of {[tuple(s) for s in shapes]}")


def _stream(x):
    return torch.cuda.current_stream(x.device)


def _c(t):
    return None if t is None else t.contiguous()


class LFilterFunction(torch.autograd.Function):
    """y, zf = filter(b, a, x, zi) for DF-II / TDF-II, fixed coefficients."""

    @staticmethod
    def forward(ctx, x, b, a, zi, form):
        _require_cuda(x, b, a, zi)
        if x.dim() != 2 or b.dim() not in (1, 2):
            raise ValueError("lfilter: x must be (B, T), b and a (M+1,) or (B, M+1)")
        Bsz, T = x.shape
        M = b.shape[-1] - 1
        coef = [(M + 1,)] if b.dim() == 1 else [(Bsz, M + 1)]
        _check(x, [("b", b, coef), ("a", a, coef), ("zi", zi, [(Bsz, M)])])
        x, b, a, zi = _c(x), _c(b), _c(a), _c(zi)
        mode = B.IIR_COEF_SHARED if b.dim() == 1 else B.IIR_COEF_PER_SEQ
        desc = B.make_desc(Bsz, T, M, form, x.dtype, mode)
        y = torch.empty_like(x)
        zf = torch.empty((Bsz, M), dtype=x.dtype, device=x.device)
        tb = B.iir_tape_bytes(desc)
        wb = B.iir_workspace_bytes(desc)
        tape = torch.empty(tb, dtype=torch.uint8, device=x.device)
        ws = torch.empty(wb, dtype=torch.uint8, device=x.device)
        with torch.cuda.device(x.device):
            B.iir_forward(desc, b, a, x, zi, y, zf, tape, tb, ws, wb, _stream(x))
        ctx.desc = desc
        ctx.save_for_backward(x, b, a, zi if zi is not None else torch.empty(0, device=x.device), y, tape)
        ctx.has_zi = zi is not None
        return y, zf

    @staticmethod
    def backward(ctx, gy, gzf):
        x, b, a, zi, y, tape = ctx.saved_tensors
        zi = zi if ctx.has_zi else None
        desc = ctx.desc
        gy = None if gy is None else _c(gy.to(x.dtype))
        gzf = None if gzf is None else _c(gzf.to(x.dtype))
        gx = torch.empty_like(x) if ctx.needs_input_grad[0] else None
        gb = torch.empty_like(b) if ctx.needs_input_grad[1] else None
        ga = torch.empty_like(a) if ctx.needs_input_grad[2] else None
        gzi = torch.empty_like(zi) if (zi is not None and ctx.needs_input_grad[3]) else None
        wb = B.iir_workspace_bytes(desc)
        ws = torch.empty(wb, dtype=torch.uint8, device=x.device)
        with torch.cuda.device(x.device):
            B.iir_backward(desc, gy, gzf, b, a, x, y, zi, tape, tape.numel(), gx, gb, ga, gzi, ws, wb, _stream(x))
        return gx, gb, ga, gzi, None


def lfilter(x, b, a, zi=None, form="tdf", return_zf=False):
    """Differentiable IIR filter of each row of x (B, T) by b, a ((M+1,) or
    (B, M+1)); zi (B, M) is the state-space initial state of the chosen form
    (TDF: scipy's zi).  Returns y, or (y, zf) when return_zf."""
    squeeze = x.dim() == 1
    if squeeze:
        x = x[None]
        zi = None if zi is None else zi[None]
    y, zf = LFilterFunction.apply(x, b, a, zi, form)
    if squeeze:
        y, zf = y[0], zf[0]
    return (y, zf) if return_zf else y


class AllPoleTVFunction(torch.autograd.Function):
    """y, zf = per-sample all-pole DF filter:
    y(n) = x(n) - sum_i a[.., n, i-1] y(n-i);  zi = [y(-1) .. y(-M)]."""

    @staticmethod
    def forward(ctx, x, a, zi):
        _require_cuda(x, a, zi)
        if x.dim() != 2 or a.dim() != 3:
            raise ValueError("allpole_tv: x must be (B, T), a (B, T, M)")
        Bsz, T = x.shape
        M = a.shape[-1]
        _check(x, [("a", a, [(Bsz, T, M)]), ("zi", zi, [(Bsz, M)])])
        x, a, zi = _c(x), _c(a), _c(zi)
        desc = B.make_desc(Bsz, T, M, "df", x.dtype, B.IIR_COEF_PER_SAMPLE)
        y = torch.empty_like(x)
        zf = torch.empty((Bsz, M), dtype=x.dtype, device=x.device)
        tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
        tape = torch.empty(tb, dtype=torch.uint8, device=x.device)
        ws = torch.empty(wb, dtype=torch.uint8, device=x.device)
        with torch.cuda.device(x.device):
            B.iir_forward(desc, None, a, x, zi, y, zf, tape, tb, ws, wb, _stream(x))
        ctx.desc = desc
        ctx.has_zi = zi is not None
        ctx.save_for_backward(a, zi if zi is not None else torch.empty(0, device=x.device), y, tape)
        return y, zf

    @staticmethod
    def backward(ctx, gy, gzf):
        a, zi, y, tape = ctx.saved_tensors
        zi = zi if ctx.has_zi else None
        desc = ctx.desc
        gx = torch.empty_like(y) if ctx.needs_input_grad[0] else None
        ga = torch.empty_like(a) if ctx.needs_input_grad[1] else None
        gzi = torch.empty_like(zi) if (zi is not None and ctx.needs_input_grad[2]) else None
        wb = B.iir_workspace_bytes(desc)
        ws = torch.empty(wb, dtype=torch.uint8, device=y.device)
        gy = None if gy is None else _c(gy.to(y.dtype))
        gzf = None if gzf is None else _c(gzf.to(y.dtype))
        with torch.cuda.device(y.device):
            B.iir_backward(desc, gy, gzf, None, a, None, y, zi, tape, tape.numel(), gx, None, ga, gzi, ws, wb,
                           _stream(y))
        return gx, ga, gzi


def allpole_tv(x, a, zi=None, return_zf=False):
    """Differentiable per-sample all-pole filter: x (B, T), a (B, T, M) with
    a[b, n, i-1] = a_i(n) (monic, a_0 = 1 implied), zi (B, M) = past outputs."""
    y, zf = AllPoleTVFunction.apply(x, a, zi)
    return (y, zf) if return_zf else y


class TVDFFunction(torch.autograd.Function):
    """y, zf = general per-sample filter.
    form "df" (R19): u(n) = x(n) - sum_i a[.., n, i-1] u(n-i),  y(n) = sum_k b[.., n, k] u(n-k);
      zi = [u(-1) .. u(-M)].
    form "tdf" (R20, the TDF realisation of PAPER.md:67-68 per sample):
      y(n) = b_0(n) x(n) + v_1(n),  v_i(n+1) = v_{i+1}(n) + b_i(n) x(n) - a_i(n) y(n);  zi = v(0)."""

    @staticmethod
    def forward(ctx, x, b, a, zi, form="df"):
        _require_cuda(x, b, a, zi)
        if x.dim() != 2 or a.dim() != 3:
            raise ValueError("lfilter_tv: x must be (B, T), b (B, T, M+1), a (B, T, M)")
        if form not in ("df", "tdf"):
            raise ValueError("lfilter_tv: form must be 'df' or 'tdf'")
        Bsz, T = x.shape
        M = a.shape[-1]
        _check(x, [("b", b, [(Bsz, T, M + 1)]), ("a", a, [(Bsz, T, M)]), ("zi", zi, [(Bsz, M)])])
        x, b, a, zi = _c(x), _c(b), _c(a), _c(zi)
        desc = B.make_desc(Bsz, T, M, form, x.dtype, B.IIR_COEF_PER_SAMPLE, flags=B.IIR_FLAG_PER_SAMPLE_B)
        y = torch.empty_like(x)
        zf = torch.empty((Bsz, M), dtype=x.dtype, device=x.device)
        tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
        tape = torch.empty(tb, dtype=torch.uint8, device=x.device)
        ws = torch.empty(wb, dtype=torch.uint8, device=x.device)
        with torch.cuda.device(x.device):
            B.iir_forward(desc, b, a, x, zi, y, zf, tape, tb, ws, wb, _stream(x))
        ctx.desc = desc
        ctx.has_zi = zi is not None
        empty = torch.empty(0, device=x.device)
        ctx.save_for_backward(b, a, zi if zi is not None else empty, y, tape, x if form == "tdf" else empty)
        ctx.form = form
        return y, zf

    @staticmethod
    def backward(ctx, gy, gzf):
        b, a, zi, y, tape, x = ctx.saved_tensors
        zi = zi if ctx.has_zi else None
        x = x if ctx.form == "tdf" else None
        desc = ctx.desc
        gx = torch.empty_like(y) if ctx.needs_input_grad[0] else None
        gb = torch.empty_like(b) if ctx.needs_input_grad[1] else None
        ga = torch.empty_like(a) if ctx.needs_input_grad[2] else None
        gzi = torch.empty_like(zi) if (zi is not None and ctx.needs_input_grad[3]) else None
        wb = B.iir_workspace_bytes(desc)
        ws = torch.empty(wb, dtype=torch.uint8, device=y.device)
        gy = None if gy is None else _c(gy.to(y.dtype))
        gzf = None if gzf is None else _c(gzf.to(y.dtype))
        with torch.cuda.device(y.device):
            B.iir_backward(desc, gy, gzf, b, a, x, y, zi, tape, tape.numel(), gx, gb, ga, gzi, ws, wb,
                           _stream(y))
        return gx, gb, ga, gzi, None


def lfilter_tv(x, b, a, zi=None, return_zf=False, form="df"):
    """Differentiable general per-sample filter: x (B, T), b (B, T, M+1), a (B, T, M)
    (a[.., n, i-1] = a_i(n), monic).  form "df": zi (B, M) = past internal signal u;
    form "tdf": the per-sample TDF-II realisation, zi = v(0) (scipy's zi for constant rows)."""
    y, zf = TVDFFunction.apply(x, b, a, zi, form)
    return (y, zf) if return_zf else y


class LTIMatrixRecurrenceFunction(torch.autograd.Function):
    """v(1..N) = recurrence(A, v0, z): v(n+1) = A v(n) + z(n) (PAPER.md:296-343,
    Listing 1), batched: z (B, N, M), v0 (B, M), A (M, M) shared or (B, M, M).
    diag=True runs the paper's Diag-EXT variant (orders 1-2)."""

    @staticmethod
    def forward(ctx, A, v0, z, diag=False):
        _require_cuda(A, v0, z)
        if z.dim() != 3 or A.dim() not in (2, 3):
            raise ValueError("matrix_recurrence: z must be (B, N, M), A (M, M) or (B, M, M)")
        Bsz, N, M = z.shape
        _check(z, [("A", A, [(M, M)] if A.dim() == 2 else [(Bsz, M, M)]), ("v0", v0, [(Bsz, M)])])
        A, v0, z = _c(A), _c(v0), _c(z)
        mode = B.IIR_COEF_SHARED if A.dim() == 2 else B.IIR_COEF_PER_SEQ
        desc = B.make_desc(Bsz, N, M, "ss", z.dtype, mode, flags=B.IIR_FLAG_DIAG if diag else 0)
        v = torch.empty_like(z)
        tb, wb = B.iir_tape_bytes(desc), B.iir_workspace_bytes(desc)
        tape = torch.empty(tb, dtype=torch.uint8, device=z.device)
        ws = torch.empty(wb, dtype=torch.uint8, device=z.device)
        with torch.cuda.device(z.device):
            B.iir_forward(desc, None, A, z, v0, v, None, tape, tb, ws, wb, _stream(z))
        ctx.desc = desc
        ctx.has_v0 = v0 is not None
        ctx.save_for_backward(A, v0 if v0 is not None else torch.empty(0, device=z.device), v, tape)
        return v

    @staticmethod
    def backward(ctx, gv):
        A, v0, v, tape = ctx.saved_tensors
        v0 = v0 if ctx.has_v0 else None
        desc = ctx.desc
        gA = torch.empty_like(A) if ctx.needs_input_grad[0] else None
        gv0 = torch.empty_like(v0) if (v0 is not None and ctx.needs_input_grad[1]) else None
        gz = torch.empty_like(v) if ctx.needs_input_grad[2] else None
        wb = B.iir_workspace_bytes(desc)
        ws = torch.empty(wb, dtype=torch.uint8, device=v.device)
        gv = None if gv is None else _c(gv.to(v.dtype))
        with torch.cuda.device(v.device):
            B.iir_backward(desc, gv, None, None, A, None, v, v0, tape, tape.numel(), gz, None, gA, gv0, ws, wb,
                           _stream(v))
        return gA, gv0, gz, None


def matrix_recurrence(A, v0, z, diag=False):
    """Differentiable batched v(n+1) = A v(n) + z(n); returns v(1..N) (B, N, M).
    diag=True: Diag-EXT (eigen-basis element-wise recursions, dense fallback for a
    defective or ill-conditioned A), orders 1 and 2."""
    return LTIMatrixRecurrenceFunction.apply(A, v0, z, diag)
