"""Host-side decode (JPEG/PNG -> HWC uint8) for the drop-in ``preprocess``.

Decode is outside the B200 hot path ("next #2"); this module
keeps the reference's observable behaviour (imgproc.py:131-260): PIL decode,
"L"/"P" promoted to RGB, any other mode rejected, and DecodeError carrying the
byte offset where the container structure first breaks.
"""

from __future__ import annotations

import io

import numpy as np
from PIL import Image, UnidentifiedImageError

from .errors import DecodeError, UnsupportedFormatError

PNG_SIGNATURE = b"\x89PNG\r\n\x1a\n"
JPEG_SOI = b"\xff\xd8"
ACCEPTED_MODES = ("L", "P", "RGB")


def _is_chunk_type(tag: bytes) -> bool:
    return len(tag) == 4 and all(chr(b).isascii() and chr(b).isalpha() for b in tag)


def png_fault_offset(data: bytes) -> int:
    """Offset of the first structural PNG fault (imgproc.py:137-163 behaviour)."""
    size = len(data)
    head = data[: len(PNG_SIGNATURE)]
    if head != PNG_SIGNATURE:
        mismatch = next((i for i, (a, b) in enumerate(zip(head, PNG_SIGNATURE)) if a != b), None)
        return size if mismatch is None else mismatch
    cursor, idat_payload = len(PNG_SIGNATURE), None
    while cursor < size:
        if size - cursor < 8:
            return cursor
        tag = data[cursor + 4: cursor + 8]
        if not _is_chunk_type(tag):
            return cursor
        if tag == b"IDAT" and idat_payload is None:
            idat_payload = cursor + 8
        nxt = cursor + 12 + int.from_bytes(data[cursor: cursor + 4], "big")
        if nxt > size:
            return size
        if tag == b"IEND":
            # chunk framing is intact, so the damage is in the compressed stream
            return cursor if idat_payload is None else idat_payload
        cursor = nxt
    return size


def jpeg_fault_offset(data: bytes) -> int:
    """Offset of the first structural JPEG fault (imgproc.py:166-196 behaviour)."""
    size = len(data)
    if data[:2] != JPEG_SOI:
        return 1 if data[:1] == b"\xff" else 0
    cursor = 2
    while cursor < size:
        if data[cursor] != 0xFF:
            return cursor
        if cursor + 1 >= size:
            return size
        code = data[cursor + 1]
        if code == 0xD9:
            return cursor  # EOI reached: the damage sits in the scan data
        if code == 0x01 or 0xD0 <= code <= 0xD7:
            cursor += 2  # parameterless markers
            continue
        if cursor + 4 > size:
            return size
        length = int.from_bytes(data[cursor + 2: cursor + 4], "big")
        if length < 2:
            return cursor + 2
        cursor += 2 + length
        if code == 0xDA:
            eoi = data.find(b"\xff\xd9", cursor)
            return size if eoi < 0 else eoi
    return size


def fault_offset(data: bytes) -> int:
    if data[:4] == PNG_SIGNATURE[:4]:
        return png_fault_offset(data)
    if data[:2] == JPEG_SOI:
        return jpeg_fault_offset(data)
    return 0


def decode_rgb(payload: bytes) -> np.ndarray:
    """Decode a JPEG or PNG payload into a C-contiguous (H, W, 3) uint8 array."""
    if not (payload[:8] == PNG_SIGNATURE or payload[:2] == JPEG_SOI):
        raise DecodeError("unrecognized image container", fault_offset(payload))
    try:
        img = Image.open(io.BytesIO(payload))
        if img.mode not in ACCEPTED_MODES:
            raise UnsupportedFormatError(f"unsupported channel layout {img.mode!r}")
        if img.mode != "RGB":
            img = img.convert("RGB")
        img.load()
        arr = np.asarray(img, dtype=np.uint8)
    except UnsupportedFormatError:
        raise
    except (UnidentifiedImageError, OSError, SyntaxError, ValueError) as exc:
        raise DecodeError(str(exc), fault_offset(payload)) from exc
    if arr.ndim == 2:
        arr = np.repeat(arr[:, :, None], 3, axis=2)
    return np.ascontiguousarray(arr)
