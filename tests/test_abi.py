"""CPU-side checks of the C ABI: the library loads, exports every symbol that
include/iirgrad.h declares, sizes workspaces, and rejects bad descriptors before
any launch (no GPU needed for any of this)."""
import ctypes
import os
import re

import pytest

from paper_2511_14390_b200 import _binding as B

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "iirgrad.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(iir_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = B.lib()
    names = declared_functions()
    assert "iir_forward" in names and "iir_backward" in names
    for n in names:
        assert hasattr(L, n), n
        assert n in B.EXPORTS, n
    assert B.iir_abi_version() == 2


def test_workspace_and_tape_sizes():
    d = B.make_desc(64, 1 << 16, 2, "tdf", B.IIR_F32, B.IIR_COEF_SHARED)
    assert B.iir_tape_bytes(d) > 0
    assert B.iir_workspace_bytes(d) > 0
    d_df = B.make_desc(64, 1 << 16, 2, "df", B.IIR_F32, B.IIR_COEF_SHARED)
    d_legacy = B.make_desc(64, 1 << 16, 2, "tdf", B.IIR_F32, B.IIR_COEF_SHARED, flags=B.IIR_FLAG_LEGACY_LTI)
    # DF keeps the state entering every 32-sample chunk (M = 2 fp32 values: 0.25 B/sample), not
    # the internal signal u (4 B/sample): the backward re-runs u from those states.
    extra = B.iir_tape_bytes(d_df) - B.iir_tape_bytes(d_legacy)
    assert 64 * (1 << 16) // 32 * 2 * 4 <= extra < 64 * (1 << 16) * 4 // 8
    # the round-2 engine's TDF tape holds only per-coefficient-set tables (no per-sample data)
    assert B.iir_tape_bytes(d) < 1 << 20
    d_seq = B.make_desc(64, 1 << 16, 8, "tdf", B.IIR_F32, B.IIR_COEF_PER_SEQ)
    assert B.iir_tape_bytes(d_seq) > B.iir_tape_bytes(B.make_desc(64, 1 << 16, 8, "tdf", B.IIR_F32, 0))


@pytest.mark.parametrize("field,value,status", [
    ("batch", 0, B.IIR_EINVAL), ("length", 0, B.IIR_EINVAL), ("order", 0, B.IIR_EUNSUPPORTED),
    ("order", 9, B.IIR_EUNSUPPORTED), ("form", 7, B.IIR_EINVAL), ("dtype", 5, B.IIR_EINVAL),
    ("coef_mode", 9, B.IIR_EINVAL)])
def test_bad_descriptor_rejected_before_launch(field, value, status):
    d = B.make_desc(2, 100, 2, "tdf", B.IIR_F32, B.IIR_COEF_SHARED)
    setattr(d, field, value)
    assert B.iir_tape_bytes(d) == 0
    L = B.lib()
    st = L.iir_forward(ctypes.byref(d), 8, 8, 8, None, 8, None, 8, 1 << 30, 8, 1 << 30, None)
    assert st == status, B.iir_last_error()
    assert len(B.iir_last_error()) > 0


def test_missing_pointers_and_small_workspace_rejected():
    d = B.make_desc(2, 100, 2, "tdf", B.IIR_F32, B.IIR_COEF_SHARED)
    L = B.lib()
    tb, wb = B.iir_tape_bytes(d), B.iir_workspace_bytes(d)
    assert L.iir_forward(ctypes.byref(d), 8, 8, None, None, 8, None, 8, tb, 8, wb, None) == B.IIR_EINVAL
    assert L.iir_forward(ctypes.byref(d), 8, 8, 8, None, 8, None, 8, tb - 1, 8, wb, None) == B.IIR_EWORKSPACE
    assert L.iir_forward(ctypes.byref(d), 8, 8, 8, None, 8, None, 8, tb, 8, wb - 1, None) == B.IIR_EWORKSPACE
    # per-sample mode is all-pole: b must be NULL
    dp = B.make_desc(2, 100, 4, "df", B.IIR_F32, B.IIR_COEF_PER_SAMPLE)
    if B.iir_tape_bytes(dp) > 0:
        assert L.iir_forward(ctypes.byref(dp), 8, 8, 8, None, 8, None, 8, 1 << 40, 8, 1 << 40, None) == B.IIR_EINVAL
    # per-sample TDF is a different filter and is not supported
    dp.form = B.IIR_TDF2
    assert B.iir_tape_bytes(dp) == 0


def test_kernel_names_and_counters():
    names = B.kernel_names()
    assert "lti_fwd" in names and "lti_bwd" in names
    assert B.iir_launch_count() >= 0


def test_state_carry_rejects_bad_arguments_before_launch():
    """iir_state_carry: argument checks return IIR_EINVAL / IIR_EUNSUPPORTED, no launch."""
    d = B.make_desc(2, 100, 2, "tdf", B.IIR_F32, B.IIR_COEF_SHARED)
    L = B.lib()
    fake = 16                                  # never dereferenced: the checks fail first
    n0 = B.iir_launch_count()
    assert L.iir_state_carry(ctypes.byref(d), fake, fake, 4, 4, 10, 0, fake, None) == B.IIR_EINVAL   # rank >= nseg
    assert L.iir_state_carry(ctypes.byref(d), fake, fake, 0, 0, 10, 0, fake, None) == B.IIR_EINVAL   # nseg < 1
    assert L.iir_state_carry(ctypes.byref(d), fake, fake, 2, 0, -1, 0, fake, None) == B.IIR_EINVAL   # seg_len < 0
    assert L.iir_state_carry(ctypes.byref(d), None, fake, 2, 0, 10, 0, fake, None) == B.IIR_EINVAL   # a NULL
    d_ss = B.make_desc(2, 100, 2, "ss", B.IIR_F32, B.IIR_COEF_SHARED)
    assert L.iir_state_carry(ctypes.byref(d_ss), fake, fake, 2, 0, 10, 0, fake, None) == B.IIR_EUNSUPPORTED
    assert B.iir_launch_count() == n0


def test_removed_three_phase_flag_rejected():
    """The three-phase LTI schedule lost on every measured shape and was removed (ABI 2)."""
    d = B.make_desc(2, 100, 2, "tdf", B.IIR_F32, B.IIR_COEF_SHARED, flags=B.IIR_FLAG_THREE_PHASE_REMOVED)
    assert B.iir_tape_bytes(d) == 0
    L = B.lib()
    assert L.iir_forward(ctypes.byref(d), 8, 8, 8, None, 8, None, 8, 1 << 30, 8, 1 << 30, None) == B.IIR_EUNSUPPORTED


def test_engine_flags_accepted_and_layouts_sized():
    """fp32 TDF: both engines have a valid tape / workspace for every order."""
    for M in range(1, 9):
        for fl in (0, B.IIR_FLAG_LEGACY_LTI, B.IIR_FLAG_ENGINE_V2, B.IIR_FLAG_GRAD_Y_EARLY):
            d = B.make_desc(3, 5000, M, "tdf", B.IIR_F32, B.IIR_COEF_SHARED, flags=fl)
            assert B.iir_tape_bytes(d) > 0 and B.iir_workspace_bytes(d) > 0, (M, fl)
