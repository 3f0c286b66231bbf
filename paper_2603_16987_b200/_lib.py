"""ctypes binding of ``libtileprep.so`` (the C-ABI in include/tileprep.h).

The library is required: importing the compute entry points without it, or
calling them without a CUDA device, raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading
from ctypes import c_int32, c_int64, c_uint64, c_void_p, c_char_p, POINTER
from pathlib import Path

import os

# TILEPREP_LIB points at an alternative build (tuning sweeps); default: the in-tree library
LIB_PATH = Path(os.environ.get("TILEPREP_LIB") or
                Path(__file__).resolve().parent / "libtileprep.so")

TP_OK = 0
TP_ERR_INVALID_ARGUMENT = 1
TP_ERR_CUDA = 2
TP_ERR_UNSUPPORTED = 3

TP_DTYPE_NONE = 0
TP_DTYPE_F32 = 1
TP_DTYPE_BF16 = 2

TP_LAYOUT_NCHW = 0
TP_LAYOUT_NHWC = 1

TP_EXPAND_ERR_MARKER_COUNT = 1
TP_EXPAND_ERR_NO_ASSISTANT = 2
TP_EXPAND_ERR_OVERFLOW = 4

TP_TILE_ALGO_AUTO = 0
TP_TILE_ALGO_FAST = 1
TP_TILE_ALGO_EXACT = 2
TP_TILE_NORM_AFFINE = 256
TP_TILE_AFTER_PLAN = 512
TP_PLAN_AFTER_KERNEL = 1
TP_PLAN_TILE_MAX_IMAGES = 4

TP_PLAN_FIELDS = 6
TP_MAX_EDGE = 65536
TP_MAX_TILES_LIMIT = 1024

_f32p = POINTER(ctypes.c_float)

# symbol -> (restype, argtypes); the order follows include/tileprep.h
SIGNATURES = {
    "tp_abi_version": (c_int32, []),
    "tp_last_error": (c_char_p, []),
    "tp_device_sm_count": (c_int32, []),
    "tp_plan": (c_int32, [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                          c_void_p]),
    "tp_plan_ex": (c_int32, [c_void_p, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
                             c_int32, c_void_p]),
    "tp_build_lut": (c_int32, [c_int32, _f32p, _f32p, c_int32, c_void_p, c_void_p]),
    "tp_lut_table_bytes": (c_int64, [c_int32, c_int32]),
    "tp_lut_bytes": (c_int64, [c_int32, c_int32]),
    "tp_build_norm": (c_int32, [c_int32, _f32p, _f32p, c_int32, c_void_p, POINTER(c_int32),
                                c_void_p]),
    "tp_tile": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p,
                          c_int32, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_int64,
                          c_void_p]),
    "tp_tile_ex": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p,
                             c_int32, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_int64,
                             c_int32, c_void_p]),
    "tp_plan_tile": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int32,
                               c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_int32,
                               c_int32, c_void_p, c_void_p, c_int64, c_int32, c_void_p]),
    "tp_plan_host": (c_int32, [c_int32, c_int32, c_int32, c_int32, c_void_p]),
    "tp_touched_rows": (c_int64, [c_int32, c_int32, c_void_p, c_void_p]),
    "tp_touched_cols": (c_int64, [c_int32, c_int32, c_void_p, c_void_p]),
    "tp_tile_rows": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p,
                               c_void_p, c_int32, c_void_p, c_int32, c_int32, c_void_p,
                               c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p]),
    "tp_host_threads": (c_int32, []),
    "tp_stage_pack": (c_int32, [c_int32, c_void_p, c_void_p, c_void_p, c_int32, c_void_p,
                                c_void_p, c_void_p, c_void_p, c_int32]),
    "tp_jpeg_parse": (c_int32, [c_void_p, c_int64, c_void_p]),
    "tp_jpeg_desc_bytes": (c_int64, []),
    "tp_jpeg_describe": (c_int64, [c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_void_p,
                                   c_void_p]),
    "tp_jpeg_decode": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_int32, c_void_p,
                                 c_int64, c_void_p, c_void_p, c_void_p]),
    "tp_png_parse": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p, c_void_p, c_int32]),
    "tp_png_desc_bytes": (c_int64, []),
    "tp_png_describe": (c_int64, [c_void_p, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "tp_png_decode": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_int64,
                                c_void_p, c_void_p, c_void_p]),
    "tp_resize": (c_int32, [c_void_p, c_int32, c_int32, c_int32, c_int32, c_int32, c_void_p,
                            c_void_p]),
    "tp_normalize": (c_int32, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_int32,
                               c_int32, c_void_p, c_void_p]),
    "tp_expand_workspace_bytes": (c_int64, [c_int32]),
    "tp_expand": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_int32, c_int32,
                            c_int32, c_int32, c_int32, c_void_p, c_int64, c_void_p, c_void_p,
                            c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "tp_supervision_mask": (c_int32, [c_void_p, c_int64, c_int64, c_int32, c_void_p, c_void_p]),
    "tp_pixel_unshuffle": (c_int32, [c_void_p, c_int32, c_int32, c_int64, c_int32, c_int32,
                                     c_void_p, c_void_p]),
    "tp_vocab_table_bytes": (c_int64, [c_int32]),
    "tp_vocab_build": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_void_p, c_void_p,
                                 c_int64]),
    "tp_tokenize_workspace_bytes": (c_int64, [c_int64, c_int32]),
    "tp_tokenize": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int64, c_void_p,
                              c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    "tp_synth": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_uint64, c_int32,
                           c_int64, c_void_p]),
}

_lock = threading.Lock()
_lib = None


class LibraryMissingError(ImportError):
    pass


def load() -> ctypes.CDLL:
    """Load (once) and type the C-ABI library; raises if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            raise LibraryMissingError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (nvcc, sm_100a). There is no CPU fallback."
            )
        lib = ctypes.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    msg = load().tp_last_error()
    return msg.decode("utf-8", "replace") if msg else ""


def check(rc: int, what: str) -> None:
    """Map a TP_* return code onto the reference's exception conventions."""
    if rc == TP_OK:
        return
    msg = last_error() or what
    if rc in (TP_ERR_INVALID_ARGUMENT, TP_ERR_UNSUPPORTED):
        raise ValueError(msg)
    from .errors import DeviceError

    raise DeviceError(f"{what}: {msg}")


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def f32_array(vals) -> ctypes.Array:
    arr = (ctypes.c_float * len(vals))()
    for i, v in enumerate(vals):
        arr[i] = float(v)
    return arr
