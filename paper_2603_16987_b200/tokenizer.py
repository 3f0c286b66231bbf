"""Drop-in placeholder expansion and supervision mask, backed by K3.

Mirrors vlmfp.tokenizer's token-sequence API (tokenizer.py:266-418):
``TokenSequence``, ``expand_image_placeholders`` and ``build_supervision_mask``
keep the reference signatures and exceptions; the splice, spans, first
assistant index and mask are computed by tp_expand / tp_supervision_mask.

``PlaceholderExpander`` is the batched device path: ragged prompt ids for a
whole batch in one launch pair, with the per-marker tile counts taken straight
from the planner's ``n_images`` tensor (no host round trip).

Greedy tokenization is K6 (tp_tokenize): ``load_vocab``
parses a vocab file with the reference's validation (tokenizer.py:72-129), the
vocabulary becomes a device hash table, and ``tokenize`` / ``tokenize_batch`` run
the longest-match walk on the GPU (tokenizer.py:135-158); ``detokenize`` is host
string work.  Any vocab object with a ``specials`` attribute naming ``image_marker``,
``image_context`` and ``assistant_header`` ids works for the expansion (the reference
``Vocab`` does), and ``load_specials`` reads those ids from a vocab file.
"""

from __future__ import annotations

import json
import re
import threading
from dataclasses import dataclass, field
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


_BYTE_TOKEN = re.compile(r"^<0x([0-9A-F]{2})>$")


@dataclass
class Vocab:
    """Immutable token table: line number (after the JSON header) = id (tokenizer.py:54-69).
    ``device_table`` caches the K6 hash table per device."""

    id_to_token: list
    token_to_id: dict
    specials: SpecialIds
    byte_ids: list  # byte value -> fallback token id, -1 when absent
    match_table: dict
    max_token_bytes: int
    _tables: dict = field(default_factory=dict, repr=False, compare=False)
    _lock: threading.Lock = field(default_factory=threading.Lock, repr=False, compare=False)

    def special_token(self, name: str) -> str:
        return self.id_to_token[getattr(self.specials, name)]

    def __len__(self) -> int:
        return len(self.id_to_token)

    def host_table(self) -> np.ndarray:
        """The K6 hash table (tp_vocab_build) as host bytes."""
        lib = _lib.load()
        items = sorted(self.match_table.items(), key=lambda kv: kv[1])
        blob = b"".join(k for k, _ in items)
        off = np.zeros(len(items) + 1, dtype=np.int32)
        off[1:] = np.cumsum([len(k) for k, _ in items])
        ids = np.asarray([i for _, i in items], dtype=np.int32)
        bids = np.asarray(self.byte_ids, dtype=np.int32)
        nbytes = lib.tp_vocab_table_bytes(len(items))
        table = np.zeros(nbytes, dtype=np.uint8)
        tok = np.frombuffer(blob, dtype=np.uint8) if blob else np.zeros(1, np.uint8)
        _lib.call("tp_vocab_build", tok.ctypes.data, off.ctypes.data, ids.ctypes.data,
                  len(items), bids.ctypes.data, table.ctypes.data, nbytes)
        return table

    def device_table(self, device) -> torch.Tensor:
        device = torch.device(device)
        with self._lock:
            t = self._tables.get(device.index)
            if t is None:
                t = torch.from_numpy(self.host_table()).to(device)
                self._tables[device.index] = t
        return t


def load_vocab(path: Union[str, Path]) -> Vocab:
    """Parse a vocab file: one JSON header line naming the special tokens, then one
    token per line, UTF-8, ids assigned in file order (tokenizer.py:72-129; same
    checks and DataError messages)."""
    return parse_vocab(Path(path).read_text(encoding="utf-8"), str(path))


def parse_vocab(raw: str, path: str = "<vocab>") -> Vocab:
    """load_vocab on the file's contents."""
    lines = raw.split("\n")
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
    id_to_token = lines[1:]
    token_to_id: dict = {}
    for i, tok in enumerate(id_to_token):
        if tok == "":
            raise DataError(f"{path}: empty token at id {i}")
        if tok in token_to_id:
            raise DataError(f"{path}: duplicate token {tok!r} at ids {token_to_id[tok]} and {i}")
        token_to_id[tok] = i
    byte_ids = [-1] * 256
    match_table: dict = {}
    max_len = 1
    for tok, i in token_to_id.items():
        m = _BYTE_TOKEN.match(tok)
        if m:
            byte_ids[int(m.group(1), 16)] = i
        else:
            b = tok.encode("utf-8")
            match_table[b] = i
            max_len = max(max_len, len(b))
    spec_map = header["specials"]
    missing = [n for n in _SPECIAL_NAMES if n not in spec_map]
    if missing:
        raise DataError(f"{path}: header missing specials {missing}")
    ids = {}
    for name in _SPECIAL_NAMES:
        tok = spec_map[name]
        if tok not in token_to_id:
            raise DataError(f"{path}: special {name}={tok!r} has no token line")
        ids[name] = token_to_id[tok]
    if len(set(ids.values())) != len(ids):
        raise DataError(f"{path}: special ids must be distinct")
    return Vocab(id_to_token=id_to_token, token_to_id=token_to_id, specials=SpecialIds(**ids),
                 byte_ids=byte_ids, match_table=match_table, max_token_bytes=max_len)


@dataclass
class TokenizedBatch:
    """Device result of tokenize_batch (int32): text t's ids are
    ids[off[t]:off[t+1]]; err[t] = 0x100 | byte when a byte has no token."""

    ids: torch.Tensor
    off: torch.Tensor
    err: torch.Tensor


@dataclass
class DeviceTexts:
    """Ragged UTF-8 texts in device memory: text t = data[off[t]:off[t+1]] (int64 off)."""

    data: torch.Tensor  # uint8 [max(total, 1)]
    off: torch.Tensor  # int64 [n + 1]
    n: int
    total: int


class DeviceTokenizer:
    """K6 with device-resident texts and reusable outputs (serving / bench path):
    ``upload`` once, then ``__call__`` enqueues the four K6 launches on a stream."""

    def __init__(self, vocab: Vocab, device=None):
        self.vocab = vocab
        self.device = require_device(device)
        self.table = vocab.device_table(self.device)
        self._ws: Optional[torch.Tensor] = None

    def upload(self, texts: Sequence) -> DeviceTexts:
        blobs = [t.encode("utf-8") if isinstance(t, str) else bytes(t) for t in texts]
        off = np.zeros(len(blobs) + 1, dtype=np.int64)
        off[1:] = np.cumsum([len(b) for b in blobs])
        total = int(off[-1])
        data = np.frombuffer(b"".join(blobs), dtype=np.uint8) if total else np.zeros(1, np.uint8)
        return DeviceTexts(torch.from_numpy(data.copy()).to(self.device),
                           torch.from_numpy(off).to(self.device), len(blobs), total)

    def alloc(self, texts: DeviceTexts) -> TokenizedBatch:
        d = self.device
        return TokenizedBatch(torch.empty(max(texts.total, 1), dtype=torch.int32, device=d),
                              torch.empty(texts.n + 1, dtype=torch.int32, device=d),
                              torch.empty(max(texts.n, 1), dtype=torch.int32, device=d))

    def __call__(self, texts: DeviceTexts, out: Optional[TokenizedBatch] = None,
                 stream: Optional[torch.cuda.Stream] = None) -> TokenizedBatch:
        out = out or self.alloc(texts)
        ws_bytes = int(_lib.load().tp_tokenize_workspace_bytes(texts.total, texts.n))
        if self._ws is None or self._ws.numel() < ws_bytes:
            self._ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            _lib.call("tp_tokenize", _lib.ptr(self.table), _lib.ptr(texts.data),
                      _lib.ptr(texts.off), texts.n, texts.total, _lib.ptr(out.ids),
                      _lib.ptr(out.off), _lib.ptr(out.err), _lib.ptr(self._ws), ws_bytes,
                      stream_handle(self.device, stream))
        return out


def tokenize_batch(texts: Sequence, vocab: Vocab, device=None,
                   stream: Optional[torch.cuda.Stream] = None) -> TokenizedBatch:
    """K6 over a batch of texts (str or UTF-8 bytes); one H2D copy of the bytes."""
    tok = DeviceTokenizer(vocab, device)
    dt = tok.upload(texts)
    res = tok(dt, stream=stream)
    return TokenizedBatch(res.ids, res.off, res.err[: dt.n])


def tokenize(text: str, vocab: Vocab) -> list:
    """Greedy longest-match over the vocabulary, byte fallback for gaps
    (tokenizer.py:135-158), on the GPU."""
    res = tokenize_batch([text], vocab)
    off = res.off.cpu().numpy()
    e = int(res.err.cpu()[0])
    if e:
        raise DataError(f"no token or byte fallback for byte 0x{e & 0xFF:02X}")
    return res.ids[off[0]: off[1]].cpu().tolist()


def detokenize(ids: list, vocab: Vocab) -> str:
    """Inverse of tokenize (tokenizer.py:161-169); host string work."""
    byte_of = {i: bytes([b]) for b, i in enumerate(vocab.byte_ids) if i >= 0}
    chunks = [byte_of[t] if t in byte_of else vocab.id_to_token[t].encode("utf-8") for t in ids]
    return b"".join(chunks).decode("utf-8")


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
        self._work = None

    def workspace(self, n_seq: int) -> torch.Tensor:
        """tp_expand's workspace (per-sequence output lengths), grown on demand."""
        nbytes = max(8, int(_lib.load().tp_expand_workspace_bytes(n_seq)))
        if self._work is None or self._work.numel() < nbytes:
            self._work = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self._work

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
                      _lib.ptr(out.mask), _lib.ptr(out.err), _lib.ptr(self.workspace(n_seq)),
                      stream_handle(d, stream))
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
