"""ctypes binding of libveckm.so (the C-ABI in include/veckm.h).

The shared library is built in-tree by `make -C paper_2504_19417_b200/csrc`
(or `__graft_entry__.build()`).  There is no CPU fallback: if the library is
missing or the device is unusable every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import DimensionMismatchError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VKM_LIB") or os.path.join(HERE, "libveckm.so")   # VKM_LIB: A/B of builds (tools)
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "veckm.h")

VKM_OK, VKM_EINVAL, VKM_EDIM, VKM_ECUDA, VKM_EOOM, VKM_EUNSUPPORTED = range(6)
MLP_MODES = {"auto": 0, "fp32": 1, "f16x3": 2, "bf16": 3}


class VkmParams(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32),
        ("delta_x", C.c_int32), ("delta_y", C.c_int32),
        ("embed_dim", C.c_int32), ("hidden", C.c_int32),
        ("delta_t", C.c_double),
        ("device", C.c_int32), ("mlp_mode", C.c_int32),
    ]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_F = C.POINTER(C.c_float)
_I32 = C.POINTER(C.c_int32)
_I64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes); every symbol declared in include/veckm.h
SIGNATURES = {
    "vkm_version": (C.c_int, []),
    "vkm_last_error": (C.c_char_p, []),
    "vkm_device_count": (C.c_int, [_I32]),
    "vkm_create": (C.c_int, [C.POINTER(_P), C.POINTER(VkmParams), _D, _D, _D, _F, _F, _F, _F]),
    "vkm_destroy": (None, [_P]),
    "vkm_set_mlp_mode": (C.c_int, [_P, C.c_int32]),
    "vkm_set_weights_f64": (C.c_int, [_P, _P, _P, _P, _P]),
    "vkm_pixel_order": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P, _P]),
    "vkm_predict_host_checked": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P, _P]),
    "vkm_predict": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P, _P]),
    "vkm_encode": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P, _P]),
    "vkm_predict_host": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P]),
    "vkm_predict_host_wide": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P]),
    "vkm_widen_f32": (C.c_int, [_P, _P, C.c_int64]),
    "vkm_concat_rows": (C.c_int, [_P, _P, C.c_int32, C.c_int64, _P]),
    "vkm_predict_multi_host": (C.c_int, [_P, C.c_int32, _P, _I64, C.c_int32, _D, _P, _P]),
    "vkm_predict_strips_host": (C.c_int, [_P, C.c_int32, _P, _P, C.c_int64, C.c_double, _P, _P]),
    "vkm_encode_host": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P]),
    "vkm_predict_f64": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P, _P]),
    "vkm_encode_f64": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P, _P]),
    "vkm_predict_f64_host": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P]),
    "vkm_encode_f64_host": (C.c_int, [_P, _P, C.c_int64, C.c_double, _P, _P]),
    "vkm_direct_encode_host": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, _P, _P]),
    "vkm_train_create": (C.c_int, [C.POINTER(_P), C.c_int32, _D, _D, C.c_int64, C.c_int32, C.c_int32, _D, _D, _D,
                                   _D, C.c_double, C.c_double, C.c_double, C.c_double]),
    "vkm_train_destroy": (None, [_P]),
    "vkm_train_epoch": (C.c_int, [_P, _P, C.c_int64, C.c_int32]),
    "vkm_train_loss": (C.c_int, [_P, _P, C.c_int64, C.POINTER(C.c_double), _I64]),
    "vkm_train_keep": (C.c_int, [_P]),
    "vkm_train_get": (C.c_int, [_P, C.c_int32, _D, _D, _D, _D]),
    "vkm_check_events": (C.c_int, [_P, C.c_int64, C.c_int64, C.c_int32, C.c_int32, _P]),
    "vkm_window_bounds": (C.c_int, [_P, _P, C.c_int64, _D, C.c_int32, C.c_double, _I64]),
    "vkm_predict_windows": (C.c_int, [_P, _P, C.c_int64, _D, _I64, C.c_int32, _P, _P, _P]),
    "vkm_predict_batch": (C.c_int, [_P, _P, _I64, C.c_int32, _D, _P, _P, _P]),
    "vkm_predict_batch_host": (C.c_int, [_P, _P, _I64, C.c_int32, _D, _P, _P]),
    "vkm_grid": (C.c_int, [_P, _P, C.c_int64, C.c_double, C.c_int32, _P, _P, _P]),
    "vkm_select_rows": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P, _I64]),
    "vkm_scatter_rows": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.c_int32, _P, _P]),
    "vkm_set_profiling": (C.c_int, [_P, C.c_int32]),
    "vkm_last_timings": (C.c_int, [_P, _F, _I32]),
}

_lib = None
_lock = threading.Lock()


def load():
    """Load libveckm.so once; raise loudly when it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `make -C {os.path.join(HERE, 'csrc')}` "
                "(the B200 path has no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    """Map a VKM_* status to the reference's exception types (errors.py:4-29)."""
    if rc == VKM_OK:
        return
    msg = load().vkm_last_error().decode(errors="replace")
    if rc == VKM_EINVAL:
        raise ValueError(msg)
    if rc == VKM_EDIM:
        raise DimensionMismatchError(msg)
    if rc == VKM_EOOM:
        raise MemoryError(msg)
    if rc == VKM_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(msg)


def declared_symbols():
    """Function names declared in include/veckm.h (for the ABI export test)."""
    import re
    with open(HEADER_PATH) as fh:
        text = fh.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(vkm_[a-z0-9_]+)\s*\(", text)))
