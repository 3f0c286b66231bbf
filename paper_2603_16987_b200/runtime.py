"""Device plumbing shared by the drop-in API and the batch engine.

PyTorch provides device memory, pinned host memory and streams; every byte of
preprocessing arithmetic runs in libtileprep.so (sm_100a).  Nothing here
computes pixels or ids on the host.
"""

from __future__ import annotations

import ctypes
import threading
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from .errors import DeviceError

_lut_lock = threading.Lock()
_lut_cache: dict[tuple, tuple] = {}


def require_device(device=None) -> torch.device:
    """The CUDA device to run on; raises DeviceError when there is none."""
    _lib.load()
    if not torch.cuda.is_available():
        raise DeviceError(
            "no CUDA device: the preprocessing path runs only on the B200 kernels "
            "(libtileprep.so); there is no CPU fallback"
        )
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    dev = torch.device(device)
    if dev.type != "cuda":
        raise DeviceError(f"device must be a CUDA device, got {dev}")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def stream_handle(device: torch.device, stream: Optional[torch.cuda.Stream] = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return s.cuda_stream


def dtype_code(tag: str) -> int:
    from .dtypes import FLOAT16_WIDE, FLOAT32

    if tag == FLOAT32:
        return _lib.TP_DTYPE_F32
    if tag == FLOAT16_WIDE:
        return _lib.TP_DTYPE_BF16
    raise ValueError(f"bad normalize_precision {tag!r}")


def torch_dtype(code: int) -> torch.dtype:
    return {_lib.TP_DTYPE_F32: torch.float32, _lib.TP_DTYPE_BF16: torch.bfloat16}[code]


def fp32_constants(vals: Sequence[float], channels: int) -> tuple[float, ...]:
    """cfg.mean[:c] rounded to fp32 exactly as np.asarray(..., float32)
    (imgproc.py:473-474); the rounding itself happens in ctypes' float cast."""
    return tuple(float(np.float32(v)) for v in tuple(vals)[:channels])


def normalize_tables(mean, std, channels: int, dtype: int,
                     device: torch.device) -> "tuple[torch.Tensor, bool]":
    """K0 via tp_build_norm: the [C,256] table (a view of a buffer that also holds the
    per-channel affine constants) and whether the affine form reproduces the table
    exactly (then K2 may normalize with one fma per value, TP_TILE_NORM_AFFINE).
    Cached per constants."""
    m = fp32_constants(mean, channels)
    s = fp32_constants(std, channels)
    if len(m) < channels or len(s) < channels:
        raise ValueError("mean/std need one entry per channel")
    key = (m, s, channels, dtype, device.index)
    with _lut_lock:
        hit = _lut_cache.get(key)
    if hit is not None:
        return hit
    lib = _lib.load()
    nbytes = lib.tp_lut_bytes(channels, dtype)
    buf = torch.empty((nbytes,), dtype=torch.uint8, device=device)
    table = buf[: channels * 256 * torch_dtype(dtype).itemsize].view(torch_dtype(dtype))
    ok = ctypes.c_int32(0)
    with torch.cuda.device(device):
        _lib.call("tp_build_norm", channels, _lib.f32_array(m), _lib.f32_array(s), dtype,
                  _lib.ptr(buf), ctypes.byref(ok), stream_handle(device))
    hit = (table.view(channels, 256), bool(ok.value))
    with _lut_lock:
        _lut_cache[key] = hit
    return hit


def normalize_lut(mean, std, channels: int, dtype: int, device: torch.device) -> torch.Tensor:
    """Device LUT [C,256] built by K0 (tp_build_norm); cached per constants."""
    return normalize_tables(mean, std, channels, dtype, device)[0]


def to_device_i32(arr, device: torch.device, non_blocking: bool = False) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int32))
    return t.to(device, non_blocking=non_blocking)


def to_device_i64(arr, device: torch.device, non_blocking: bool = False) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.int64))
    return t.to(device, non_blocking=non_blocking)
