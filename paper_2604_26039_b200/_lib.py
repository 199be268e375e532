"""ctypes binding of libramp_b200.so (the C ABI in include/ramp_b200.h).

There is deliberately no CPU fallback: if the library or an sm_100a device is
missing, every call raises.  `load()` is the single place the .so is opened.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libramp_b200.so"

c_i32p = ctypes.POINTER(ctypes.c_int32)

# Every symbol include/ramp_b200.h declares, with (restype, argtypes).
SIGNATURES = {
    "ramp_version": (ctypes.c_int, []),
    "ramp_set_profile_buffer": (None, [ctypes.c_void_p]),
    "ramp_last_error": (ctypes.c_char_p, []),
    "ramp_device_ok": (ctypes.c_int, []),
    "ramp_align_capacity": (ctypes.c_int64, [ctypes.c_int64, ctypes.c_int32, ctypes.c_int32]),
    "ramp_config_smem_bytes": (ctypes.c_int64, [ctypes.c_int32] * 4),
    "ramp_moe_align": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    ),
    "ramp_dispatch_select": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p],
    ),
    "ramp_fused_moe_workspace_size": (ctypes.c_size_t, [ctypes.c_int32] * 5),
    "ramp_fused_moe_bf16": (
        ctypes.c_int,
        [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
         ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
         ctypes.c_size_t, ctypes.c_void_p],
    ),
}
SIGNATURES["ramp_config_smem_bytes_fp8"] = (ctypes.c_int64, [ctypes.c_int32] * 3)
SIGNATURES["ramp_config_smem_bytes_fp8_kps"] = (ctypes.c_int64, [ctypes.c_int32] * 4)
SIGNATURES["ramp_config_smem_bytes_kps"] = (ctypes.c_int64, [ctypes.c_int32] * 5)
SIGNATURES["ramp_fused_moe_gating_bf16"] = (
    ctypes.c_int,
    [ctypes.c_void_p] * 4 + [ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
    + [ctypes.c_int32] * 5 + [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                              ctypes.c_size_t, ctypes.c_void_p])
SIGNATURES["ramp_fused_moe_fp8"] = (
    ctypes.c_int,
    [ctypes.c_void_p] * 7 + [ctypes.c_int32] * 5 + [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                                    ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32, ctypes.c_void_p])
SIGNATURES["ramp_fused_moe_fp8_prequant"] = (
    ctypes.c_int,
    [ctypes.c_void_p] * 8 + [ctypes.c_int32] * 5 + [ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                                    ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32, ctypes.c_void_p])
_vp, _i32 = ctypes.c_void_p, ctypes.c_int32
SIGNATURES["ramp_fused_moe_strided"] = (
    ctypes.c_int, [_vp] * 9 + [_i32] * 5 + [_vp, _i32, _vp, _vp, _vp, ctypes.c_size_t, _i32, _vp])
SIGNATURES["ramp_ep_row_layout"] = (ctypes.c_int, [_i32] * 3 + [_vp])
SIGNATURES["ramp_ep_pack"] = (ctypes.c_int, [_vp] * 3 + [_i32] * 7 + [_vp] * 5)
SIGNATURES["ramp_ep_reduce"] = (ctypes.c_int, [_vp, _vp] + [_i32] * 4 + [_vp, _vp])
SIGNATURES["ramp_ep_get_unique_id"] = (ctypes.c_int, [_vp])
SIGNATURES["ramp_ep_comm_init"] = (ctypes.c_int, [ctypes.POINTER(_vp), _vp, _i32, _i32])
SIGNATURES["ramp_ep_comm_destroy"] = (ctypes.c_int, [_vp])
SIGNATURES["ramp_ep_dispatch"] = (ctypes.c_int, [_vp] * 4 + [_i32] * 6 + [_vp] * 6)
SIGNATURES["ramp_ep_combine"] = (ctypes.c_int, [_vp] * 4 + [_i32] * 3 + [_vp, _vp])
SIGNATURES["ramp_fused_moe_bf16_ex"] = (
    ctypes.c_int, SIGNATURES["ramp_fused_moe_bf16"][1][:-1] + [ctypes.c_int32, ctypes.c_void_p])


class RampTable(ctypes.Structure):
    """Mirror of `ramp_table_t`: device pointers + geometry scalars."""

    _fields_ = [
        ("n_cfg", ctypes.c_int32),
        ("n_ubm", ctypes.c_int32),
        ("N", ctypes.c_int32),
        ("kappa_ok", ctypes.c_int32),
        ("sm_count", ctypes.c_int32),
        ("reserved", ctypes.c_int32 * 3),
        ("bm", ctypes.c_void_p),
        ("ttn", ctypes.c_void_p),
        ("stg", ctypes.c_void_p),
        ("split_k", ctypes.c_void_p),
        ("group_m", ctypes.c_void_p),
        ("mode", ctypes.c_void_p),
        ("ubm", ctypes.c_void_p),
        ("ubm_index", ctypes.c_void_p),
        ("a", ctypes.c_void_p),
        ("b", ctypes.c_void_p),
        ("c", ctypes.c_void_p),
        ("d", ctypes.c_void_p),
        ("ntile", ctypes.c_void_p),
        ("omega_max", ctypes.c_double),
        ("lam", ctypes.c_void_p),
        ("kps", ctypes.c_void_p),
        ("step_cache", ctypes.c_void_p),
        ("step_cache_cap", ctypes.c_int32),
        ("h3", ctypes.c_void_p),
    ]


class RowStrides(ctypes.Structure):
    """ramp_row_strides_t (include/ramp_b200.h): token-row strides, 0 = dense."""

    _fields_ = [("x_stride", ctypes.c_int64), ("sf_stride", ctypes.c_int64), ("ids_stride", ctypes.c_int64),
                ("w_stride", ctypes.c_int64)]


class RampError(RuntimeError):
    pass


_lib = None


def load() -> ctypes.CDLL:
    """Open libramp_b200.so (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is None:
        path = os.environ.get("RAMP_B200_LIB", str(LIB_PATH))
        if not Path(path).exists():
            raise RampError(
                f"{path} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        lib = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = load().ramp_last_error().decode(errors="replace")
        if rc == 1:
            raise ValueError(msg)
        raise RampError(f"libramp_b200 error {rc}: {msg}")


def require_device() -> None:
    if not load().ramp_device_ok():
        raise RampError("libramp_b200 needs an sm_100 (B200) GPU; none is visible")
