"""ctypes binding of libiirgrad.so (include/iirgrad.h) -- argument marshalling only.

Every function here has the name of the C entry point it wraps.  Tensors are
passed by their device pointer; ``None`` becomes NULL.  All arithmetic runs in
the library's CUDA kernels; if the library is missing this module raises at
load time -- there is no fallback.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IIRG_LIB") or os.path.join(HERE, "lib", "libiirgrad.so")   # IIRG_LIB: build variants

IIR_OK, IIR_EINVAL, IIR_EUNSUPPORTED, IIR_ECUDA, IIR_EWORKSPACE = range(5)
IIR_DF2, IIR_TDF2, IIR_SS = 0, 1, 2
IIR_F32, IIR_F64 = 0, 1
IIR_COEF_SHARED, IIR_COEF_PER_SEQ, IIR_COEF_PER_SAMPLE = 0, 1, 2
IIR_FLAG_WS_READY = 1
IIR_FLAG_SINGLE_PASS = 2
IIR_FLAG_THREE_PHASE_REMOVED = 4
IIR_FLAG_PER_SAMPLE_B = 8
IIR_FLAG_LEGACY_LTI = 16
IIR_FLAG_ENGINE_V2 = 32
IIR_FLAG_GRAD_Y_EARLY = 64
IIR_FLAG_DIAG = 128

FORMS = {"df": IIR_DF2, "tdf": IIR_TDF2, "ss": IIR_SS, IIR_DF2: IIR_DF2, IIR_TDF2: IIR_TDF2, IIR_SS: IIR_SS}
DTYPES = {torch.float32: IIR_F32, torch.float64: IIR_F64}

EXPORTS = ["iir_tape_bytes", "iir_workspace_bytes", "iir_workspace_init", "iir_forward", "iir_backward", "iir_last_error",
           "iir_abi_version", "iir_launch_count", "iir_num_kernels", "iir_kernel_name",
           "iir_profile_enable", "iir_profile_reset", "iir_profile_query", "iir_debug_trace", "iir_state_carry",
           "iir_check_workspace"]


class Desc(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int64), ("length", ctypes.c_int64), ("order", ctypes.c_int32),
                ("form", ctypes.c_int32), ("dtype", ctypes.c_int32), ("coef_mode", ctypes.c_int32),
                ("flags", ctypes.c_int32)]

    def __repr__(self):
        return (f"Desc(batch={self.batch}, length={self.length}, order={self.order}, form={self.form}, "
                f"dtype={self.dtype}, coef_mode={self.coef_mode}, flags={self.flags})")


class IIRError(RuntimeError):
    pass


_lib = None
_lock = threading.Lock()
_vp = ctypes.c_void_p


def lib():
    """Load libiirgrad.so (once).  Raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise IIRError(f"{LIB_PATH} not found: build it with `python -m paper_2511_14390_b200.build` "
                           "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        dp = ctypes.POINTER(Desc)
        L.iir_tape_bytes.restype = ctypes.c_size_t
        L.iir_tape_bytes.argtypes = [dp]
        L.iir_workspace_bytes.restype = ctypes.c_size_t
        L.iir_workspace_bytes.argtypes = [dp]
        L.iir_workspace_init.restype = ctypes.c_int
        L.iir_workspace_init.argtypes = [dp, _vp, ctypes.c_size_t, _vp]
        L.iir_forward.restype = ctypes.c_int
        L.iir_forward.argtypes = [dp] + [_vp] * 7 + [ctypes.c_size_t, _vp, ctypes.c_size_t, _vp]
        L.iir_backward.restype = ctypes.c_int
        L.iir_backward.argtypes = [dp] + [_vp] * 8 + [ctypes.c_size_t] + [_vp] * 5 + [ctypes.c_size_t, _vp]
        L.iir_state_carry.restype = ctypes.c_int
        L.iir_state_carry.argtypes = [dp, _vp, _vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32,
                                      _vp, _vp]
        L.iir_check_workspace.restype = ctypes.c_int
        L.iir_check_workspace.argtypes = [dp, _vp, ctypes.c_size_t, _vp]
        L.iir_last_error.restype = ctypes.c_char_p
        L.iir_abi_version.restype = ctypes.c_int
        L.iir_launch_count.restype = ctypes.c_int64
        L.iir_num_kernels.restype = ctypes.c_int
        L.iir_kernel_name.restype = ctypes.c_char_p
        L.iir_kernel_name.argtypes = [ctypes.c_int]
        L.iir_profile_enable.argtypes = [ctypes.c_int]
        L.iir_debug_trace.argtypes = [_vp]
        L.iir_profile_query.restype = ctypes.c_int
        L.iir_profile_query.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
        _lib = L
        return L


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def _check(status, what):
    if status != IIR_OK:
        msg = lib().iir_last_error().decode()
        raise IIRError(f"{what} failed with status {status}: {msg}")


def make_desc(batch, length, order, form="tdf", dtype=torch.float32, coef_mode=IIR_COEF_SHARED, flags=0) -> Desc:
    return Desc(int(batch), int(length), int(order), FORMS[form],
                DTYPES[dtype] if isinstance(dtype, torch.dtype) else int(dtype), int(coef_mode), int(flags))


def iir_tape_bytes(desc: Desc) -> int:
    return lib().iir_tape_bytes(ctypes.byref(desc))


def iir_workspace_bytes(desc: Desc) -> int:
    return lib().iir_workspace_bytes(ctypes.byref(desc))


def iir_workspace_init(desc, ws, ws_bytes, stream=None):
    _check(lib().iir_workspace_init(ctypes.byref(desc), _ptr(ws), int(ws_bytes), _stream(stream)),
           "iir_workspace_init")


def _stream(stream):
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def iir_forward(desc, b, a, x, zi, y, zf, tape, tape_bytes, ws, ws_bytes, stream=None):
    st = lib().iir_forward(ctypes.byref(desc), _ptr(b), _ptr(a), _ptr(x), _ptr(zi), _ptr(y), _ptr(zf),
                           _ptr(tape), int(tape_bytes), _ptr(ws), int(ws_bytes), _stream(stream))
    _check(st, "iir_forward")


def iir_backward(desc, grad_y, grad_zf, b, a, x, y, zi, tape, tape_bytes, grad_x, grad_b, grad_a, grad_zi,
                 ws, ws_bytes, stream=None):
    st = lib().iir_backward(ctypes.byref(desc), _ptr(grad_y), _ptr(grad_zf), _ptr(b), _ptr(a), _ptr(x), _ptr(y),
                            _ptr(zi), _ptr(tape), int(tape_bytes), _ptr(grad_x), _ptr(grad_b), _ptr(grad_a),
                            _ptr(grad_zi), _ptr(ws), int(ws_bytes), _stream(stream))
    _check(st, "iir_backward")


def iir_state_carry(desc, a, w, nseg, rank, seg_len, reverse, out, stream=None):
    st = lib().iir_state_carry(ctypes.byref(desc), _ptr(a), _ptr(w), int(nseg), int(rank), int(seg_len),
                               1 if reverse else 0, _ptr(out), _stream(stream))
    _check(st, "iir_state_carry")


def iir_check_workspace(desc, ws, ws_bytes, stream=None):
    """Synchronise and raise if a look-back wait of the last call on ws timed out."""
    _check(lib().iir_check_workspace(ctypes.byref(desc), _ptr(ws), int(ws_bytes), _stream(stream)),
           "iir_check_workspace")


def iir_last_error() -> str:
    return lib().iir_last_error().decode()


def iir_abi_version() -> int:
    return lib().iir_abi_version()


def iir_launch_count() -> int:
    return lib().iir_launch_count()


def kernel_names():
    L = lib()
    return [L.iir_kernel_name(k).decode() for k in range(L.iir_num_kernels())]


def iir_profile_enable(on: bool):
    lib().iir_profile_enable(1 if on else 0)


def iir_profile_reset():
    lib().iir_profile_reset()


def iir_profile_query(kind: int):
    ms = ctypes.c_double()
    n = ctypes.c_int64()
    lib().iir_profile_query(int(kind), ctypes.byref(ms), ctypes.byref(n))
    return ms.value, n.value


def iir_debug_trace(buf):
    lib().iir_debug_trace(_ptr(buf))
