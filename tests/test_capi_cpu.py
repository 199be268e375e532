"""The C-ABI library loads without a GPU, exports every symbol the public
header declares, and validates arguments before touching the device."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from paper_2604_26039_b200 import _lib
from paper_2604_26039_b200.config_space import B200_SMEM_LIMIT, b200_smem_bytes

HEADER = Path(__file__).resolve().parents[1] / "include" / "ramp_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ramp_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    return _lib.load()


def test_every_declared_symbol_is_exported(lib):
    syms = declared_symbols()
    assert len(syms) >= 9
    for s in syms:
        assert hasattr(lib, s), s
        assert s in _lib.SIGNATURES, f"{s} has no ctypes signature"


def test_version_and_capacity(lib):
    assert lib.ramp_version() >= 100
    assert lib.ramp_align_capacity(8, 64, 16) == ((8 + 64 * 15 + 15) // 16) * 16
    assert lib.ramp_align_capacity(-1, 64, 16) == 0


def test_smem_formula_matches_python(lib):
    for bm in (4, 8, 16, 32, 64, 128):
        for ttn in (128, 256, 512):
            for stg in range(1, 13):
                for mode in (0, 1):
                    want = b200_smem_bytes(bm, ttn, stg, mode)
                    got = lib.ramp_config_smem_bytes(bm, ttn, stg, mode)
                    assert got == (want if want <= B200_SMEM_LIMIT else 0), (bm, ttn, stg, mode)
    assert lib.ramp_config_smem_bytes(4, 384, 2, 0) == 0
    for bm in (4, 16, 32):
        for ttn in (128, 256):
            for stg in range(1, 13):
                for mode in (0, 1):
                    for kps in (1, 2, 4):
                        want = b200_smem_bytes(bm, ttn, stg, mode, kps)
                        got = lib.ramp_config_smem_bytes_kps(bm, ttn, stg, mode, kps)
                        assert got == (want if want <= B200_SMEM_LIMIT else 0), (bm, ttn, stg, mode, kps)
    assert lib.ramp_config_smem_bytes_kps(16, 128, 2, 1, 3) == 0


def test_argument_validation_without_gpu(lib):
    buf = (ctypes.c_int32 * 16)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    rc = lib.ramp_moe_align(p, 8, 0, 16, p, p, p, p, None)
    assert rc == 1 and b"E must be" in lib.ramp_last_error()
    rc = lib.ramp_moe_align(p, 8, 64, 0, p, p, p, p, None)
    assert rc == 1 and b"bm must be" in lib.ramp_last_error()
    rc = lib.ramp_dispatch_select(p, 64, None, p, p, None, None, None)
    assert rc == 1 and b"table is null" in lib.ramp_last_error()
    t = _lib.RampTable()
    rc = lib.ramp_dispatch_select(p, 64, ctypes.byref(t), p, p, None, None, None)
    assert rc == 1 and b"empty pool" in lib.ramp_last_error()
    with pytest.raises(ValueError):
        _lib.check(1)


def test_no_device_reported(lib):
    import torch

    if not torch.cuda.is_available():
        assert lib.ramp_device_ok() == 0


def test_ep_argument_validation_without_gpu(lib):
    """The expert-parallel entry points reject bad geometry before any launch."""
    buf = (ctypes.c_int32 * 64)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    # world must divide E
    rc = lib.ramp_ep_pack(p, p, p, 4, 128, 10, 2, 4, 4, 0, p, p, p, p, None)
    assert rc == 1 and b"multiple of world" in lib.ramp_last_error()
    rc = lib.ramp_ep_pack(p, p, p, 4, 100, 8, 2, 4, 4, 0, p, p, p, p, None)
    assert rc == 1 and b"H (d_model)" in lib.ramp_last_error()
    rc = lib.ramp_ep_pack(p, p, p, 4, 128, 8, 2, 4, 4, 7, p, p, p, p, None)
    assert rc == 1 and b"wire" in lib.ramp_last_error()
    rc = lib.ramp_ep_pack(p, p, p, 4, 128, 8, 2, 4, 4, 1, None, p, p, p, None)
    assert rc == 1 and b"null send buffer" in lib.ramp_last_error()
    rc = lib.ramp_ep_reduce(p, p, 4, 128, 0, 4, p, None)
    assert rc == 1
    rc = lib.ramp_ep_dispatch(None, p, p, p, 4, 128, 8, 2, 4, 0, p, p, p, p, p, None)
    assert rc == 1 and b"communicator" in lib.ramp_last_error()
    comm = ctypes.c_void_p()
    rc = lib.ramp_ep_comm_init(ctypes.byref(comm), p, 0, 0)
    assert rc == 1 and b"world" in lib.ramp_last_error()


def test_ep_row_layout_matches_python_and_oracle(lib):
    """ramp_ep_row_layout, ep.row_layout and the oracle's restatement agree."""
    from oracle.ep_ref import row_layout_ref
    from paper_2604_26039_b200.ep import row_layout

    out = (ctypes.c_int32 * 4)()
    for H in (128, 384, 2048, 7168):
        for k in (1, 2, 3, 8):
            for wire, code in (("bf16", 0), ("fp8", 1)):
                assert lib.ramp_ep_row_layout(H, k, code, out) == 0
                got = tuple(out)
                assert got == row_layout_ref(H, k, wire) == tuple(vars(row_layout(H, k, wire)).values())
                assert got[1] % 16 == 0 and got[3] % 16 == 0
    assert lib.ramp_ep_row_layout(100, 2, 0, out) == 1


def test_strided_entry_validation_without_gpu(lib):
    """ramp_fused_moe_strided rejects malformed strides before any launch."""
    buf = (ctypes.c_int32 * 64)()
    p = ctypes.cast(buf, ctypes.c_void_p)
    t = _lib.RampTable()
    st = _lib.RowStrides(100, 0, 0, 0)  # not a multiple of 16
    rc = lib.ramp_fused_moe_strided(p, None, p, None, p, None, p, p, ctypes.byref(st), 4, 128, 128, 8, 2,
                                    ctypes.byref(t), -1, p, None, p, 1 << 20, 3, None)
    assert rc == 1 and b"x_stride" in lib.ramp_last_error()
    st = _lib.RowStrides(0, 0, 1, 0)  # ids_stride below top_k
    rc = lib.ramp_fused_moe_strided(p, None, p, None, p, None, p, p, ctypes.byref(st), 4, 128, 128, 8, 2,
                                    ctypes.byref(t), -1, p, None, p, 1 << 20, 3, None)
    assert rc == 1 and b"ids_stride" in lib.ramp_last_error()
