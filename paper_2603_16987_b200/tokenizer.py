"""Drop-in placeholder expansion and supervision mask, backed by K3.

Mirrors vlmfp.tokenizer's token-sequence API (tokenizer.py:266-418):
``TokenSequence``, ``expand_image_placeholders`` and ``build_supervision_mask``
keep the reference signatures and exceptions; the splice, spans, first
assistant index and mask are computed by tp_expand / tp_supervision_mask.

``PlaceholderExpander`` is the batched device path: ragged prompt ids for a
whole batch in one launch pair, with the per-marker tile counts taken straight
from the planner's ``n_images`` tensor (no host round trip).

Vocabulary loading and greedy tokenization stay out of scope;
any vocab object with a ``specials`` attribute naming ``image_marker``,
``image_context`` and ``assistant_header`` ids works (the reference ``Vocab``
does), and ``load_specials`` reads those ids from a vocab file.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Sequence, Union

import numpy as np
import torch

from . import _lib
from .errors import DataError, ExpansionError, MalformedSequenceError
from .runtime import require_device, stream_handle

_SPECIAL_NAMES = ("bos", "eos", "user_header", "assistant_header", "image_marker",
                  "image_context", "pad")


@dataclass(frozen=True)
class SpecialIds:
    """Special-token ids (tokenizer.py:43-51)."""

    bos: int
    eos: int
    user_header: int
    assistant_header: int
    image_marker: int
    image_context: int
    pad: int


@dataclass
class SpecialVocab:
    """Minimal vocab stand-in: only the specials the hot path needs."""

    specials: SpecialIds


def load_specials(path: Union[str, Path]) -> SpecialVocab:
    """Special ids of a vocab file: JSON header naming the specials, then one
    token per line, id = line index (format of tokenizer.py:72-129)."""
    lines = Path(path).read_text(encoding="utf-8").split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    if not lines:
        raise DataError(f"{path}: empty vocab file")
    try:
        header = json.loads(lines[0])
    except json.JSONDecodeError as exc:
        raise DataError(f"{path}: bad JSON header: {exc}") from exc
    if not isinstance(header, dict) or "specials" not in header:
        raise DataError(f"{path}: header must be an object with a 'specials' map")
    index = {}
    for i, tok in enumerate(lines[1:]):
        index.setdefault(tok, i)
    ids = {}
    for name in _SPECIAL_NAMES:
        tok = header["specials"].get(name)
        if tok is None or tok not in index:
            raise DataError(f"{path}: special {name}={tok!r} has no token line")
        ids[name] = index[tok]
    if len(set(ids.values())) != len(ids):
        raise DataError(f"{path}: special ids must be distinct")
    return SpecialVocab(SpecialIds(**ids))


@dataclass
class TokenSequence:
    """Ids plus the supervision bookkeeping for the masked loss (tokenizer.py:266-291)."""

    ids: list[int]
    first_assistant_index: int
    image_spans: list[tuple[int, int]]
    supervision_mask: list[bool]

    def validate(self, vocab) -> "TokenSequence":
        T = len(self.ids)
        if not 0 <= self.first_assistant_index <= T:
            raise MalformedSequenceError(
                f"first_assistant_index {self.first_assistant_index} outside [0, {T}]"
            )
        if len(self.supervision_mask) != T:
            raise MalformedSequenceError("mask length != sequence length")
        if self.image_spans:
            ids = np.asarray(self.ids, dtype=np.int64)
            ctx = vocab.specials.image_context
            for start, length in self.image_spans:
                if start < 0 or length < 1 or start + length > T:
                    raise MalformedSequenceError(f"image span ({start}, {length}) out of range")
                if np.any(ids[start: start + length] != ctx):
                    raise MalformedSequenceError(
                        f"image span ({start}, {length}) covers non-placeholder ids"
                    )
        return self


@dataclass
class ExpandedBatch:
    """Device result of a batched expansion (all int32 unless noted)."""

    ids: torch.Tensor  # [capacity] expanded ids, sequence s at out_off[s]:out_off[s+1]
    out_off: torch.Tensor  # [n_seq + 1]; out_off[-1] == -1 on capacity overflow
    spans: torch.Tensor  # [n_markers, 2] (start, length) relative to the sequence
    first_assistant: torch.Tensor  # [n_seq], -1 when absent
    mask: torch.Tensor  # uint8 [capacity]
    err: torch.Tensor  # [n_seq] TP_EXPAND_ERR_* flags


class PlaceholderExpander:
    """Batched image-placeholder expansion on device (K3)."""

    def __init__(self, vocab, tokens_per_tile: int, device=None, with_mask: bool = True):
        sp = vocab.specials
        self.marker = int(sp.image_marker)
        self.ctx = int(sp.image_context)
        self.asst = int(sp.assistant_header)
        if tokens_per_tile < 0:
            raise ValueError("tokens_per_tile must be >= 0")
        self.tpt = int(tokens_per_tile)
        self.with_mask = with_mask
        self.device = require_device(device)

    def __call__(self, ids: torch.Tensor, seq_off: torch.Tensor, counts: torch.Tensor,
                 count_off: torch.Tensor, capacity: int, out: Optional[ExpandedBatch] = None,
                 stream: Optional[torch.cuda.Stream] = None) -> ExpandedBatch:
        n_seq = seq_off.numel() - 1
        n_cnt = counts.numel()
        d = self.device
        if out is None:
            out = ExpandedBatch(
                ids=torch.empty((max(capacity, 1),), dtype=torch.int32, device=d),
                out_off=torch.empty((n_seq + 1,), dtype=torch.int32, device=d),
                spans=torch.empty((max(n_cnt, 1), 2), dtype=torch.int32, device=d),
                first_assistant=torch.empty((max(n_seq, 1),), dtype=torch.int32, device=d),
                mask=torch.empty((max(capacity, 1),), dtype=torch.uint8, device=d),
                err=torch.empty((max(n_seq, 1),), dtype=torch.int32, device=d),
            )
        with torch.cuda.device(d):
            _lib.call("tp_expand", _lib.ptr(ids), _lib.ptr(seq_off), n_seq, _lib.ptr(counts),
                      _lib.ptr(count_off), self.tpt, self.marker, self.ctx, self.asst,
                      1 if self.with_mask else 0, _lib.ptr(out.ids), capacity,
                      _lib.ptr(out.out_off), _lib.ptr(out.spans), _lib.ptr(out.first_assistant),
                      _lib.ptr(out.mask), _lib.ptr(out.err), None, stream_handle(d, stream))
        return out


def _raise_for(flags: int, n_markers: int, n_counts: int) -> None:
    if flags & _lib.TP_EXPAND_ERR_MARKER_COUNT:
        raise ExpansionError(f"{n_markers} markers but {n_counts} tile counts")
    if flags & _lib.TP_EXPAND_ERR_OVERFLOW:
        raise ValueError("expanded sequence length is negative or exceeds int32")
    if flags & _lib.TP_EXPAND_ERR_NO_ASSISTANT:
        raise MalformedSequenceError("sequence has no assistant header")


def expand_image_placeholders(ids: list[int], counts: list[int], tokens_per_tile: int,
                              vocab) -> TokenSequence:
    """Replace each image-marker id with tiles * tokens_per_tile context ids
    (tokenizer.py:294-315); the mask is all False, as in the reference."""
    return _expand_one(ids, counts, tokens_per_tile, vocab, with_mask=False)


def _expand_one(ids: Sequence[int], counts: Sequence[int], tokens_per_tile: int, vocab,
                with_mask: bool) -> TokenSequence:
    exp = PlaceholderExpander(vocab, tokens_per_tile, with_mask=with_mask)
    d = exp.device
    ids_np = np.asarray(list(ids), dtype=np.int32)
    cnt_np = np.asarray(list(counts), dtype=np.int64)
    n_markers = int(np.count_nonzero(ids_np == exp.marker))
    if n_markers != len(cnt_np):  # the reference checks this before anything else
        raise ExpansionError(f"{n_markers} markers but {len(cnt_np)} tile counts")
    cap = int(len(ids_np) + max(0, int((cnt_np * tokens_per_tile).sum())))
    ids_t = torch.from_numpy(ids_np).to(d)
    cnt_t = torch.from_numpy(cnt_np.astype(np.int32)).to(d)
    seq_off = torch.tensor([0, len(ids_np)], dtype=torch.int32, device=d)
    count_off = torch.tensor([0, len(cnt_np)], dtype=torch.int32, device=d)
    res = exp(ids_t, seq_off, cnt_t, count_off, cap)
    err = int(res.err[0].item())
    _raise_for(err, n_markers, len(cnt_np))
    n = int(res.out_off[1].item())
    out_ids = res.ids[:n].cpu().tolist()
    spans = [(int(a), int(b)) for a, b in res.spans[: len(cnt_np)].cpu().tolist()]
    t = int(res.first_assistant[0].item())
    mask = res.mask[:n].cpu().numpy().astype(bool).tolist() if with_mask else [False] * n
    return TokenSequence(out_ids, t, spans, mask)


def build_supervision_mask(seq: TokenSequence, vocab) -> TokenSequence:
    """Mark assistant response tokens: index >= t, header ids excluded
    (tokenizer.py:410-418), then validate."""
    T = len(seq.ids)
    t = seq.first_assistant_index
    if not 0 <= t <= T:
        raise MalformedSequenceError(f"first_assistant_index {t} outside [0, {T}]")
    device = require_device()
    if T:
        ids = torch.from_numpy(np.asarray(seq.ids, dtype=np.int32)).to(device)
        mask = torch.empty((T,), dtype=torch.uint8, device=device)
        _lib.call("tp_supervision_mask", _lib.ptr(ids), T, t,
                  int(vocab.specials.assistant_header), _lib.ptr(mask), stream_handle(device))
        mask_list = mask.cpu().numpy().astype(bool).tolist()
    else:
        mask_list = []
    return TokenSequence(seq.ids, t, seq.image_spans, mask_list).validate(vocab)


def expand_and_mask(ids: list[int], counts: list[int], tokens_per_tile: int,
                    vocab) -> TokenSequence:
    """expand_image_placeholders followed by build_supervision_mask in one K3
    pass (the compact path of build_token_sequence, tokenizer.py:388-407)."""
    seq = _expand_one(ids, counts, tokens_per_tile, vocab, with_mask=True)
    return seq.validate(vocab)


__all__ = [
    "ExpandedBatch",
    "PlaceholderExpander",
    "SpecialIds",
    "SpecialVocab",
    "TokenSequence",
    "build_supervision_mask",
    "expand_and_mask",
    "expand_image_placeholders",
    "load_specials",
]
