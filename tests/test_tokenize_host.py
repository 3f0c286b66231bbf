"""Vocabulary loading and the K6 hash table, on the host (CPU).

load_vocab re-expresses the reference's checks (vlmfp tests/test_tokenizer.py:100-124);
the table built by tp_vocab_build (host C code in libtileprep.so) is walked here with a
Python restatement of K6's probe sequence and must reproduce the reference's ids for
every golden text, which pins the table layout and hash the GPU kernel uses.
"""

from __future__ import annotations

import json
import struct

import numpy as np
import pytest

from oracle import tileprep_oracle as O
from paper_2603_16987_b200 import _lib
from paper_2603_16987_b200.errors import DataError
from paper_2603_16987_b200.tokenizer import detokenize, load_vocab

HEADER = {"specials": {"bos": "<b>", "eos": "<e>", "user_header": "<u>",
                       "assistant_header": "<a>", "image_marker": "<i>",
                       "image_context": "<c>", "pad": "<p>"}}
SPECIALS = ["<b>", "<e>", "<u>", "<a>", "<i>", "<c>", "<p>"]


def write_vocab(tmp_path, tokens, header=None):
    path = tmp_path / "vocab.txt"
    path.write_text(json.dumps(header or HEADER) + "\n" + "\n".join(SPECIALS + tokens) + "\n",
                    encoding="utf-8")
    return path


@pytest.fixture(scope="module")
def golden_vocab(tmp_path_factory, golden):
    _, meta = golden
    path = tmp_path_factory.mktemp("v") / "base_vocab.txt"
    path.write_text(meta["vocab_file"], encoding="utf-8")
    return load_vocab(path), meta


def test_golden_vocab_parses(golden_vocab):
    vocab, meta = golden_vocab
    toks, bids, table, max_len = O.parse_vocab(meta["vocab_file"])
    assert vocab.id_to_token == toks and vocab.byte_ids == bids
    assert vocab.match_table == table and vocab.max_token_bytes == max_len == 13
    assert vocab.specials.image_marker == meta["specials"]["image_marker"]


def test_load_vocab_rejects_bad_files(tmp_path):
    with pytest.raises(DataError):
        load_vocab(write_vocab(tmp_path, ["a", "a"]))
    with pytest.raises(DataError):
        load_vocab(write_vocab(tmp_path, ["a"], {"specials": {"bos": "<b>"}}))
    bad = tmp_path / "bad.txt"
    bad.write_text("not json\na\n", encoding="utf-8")
    with pytest.raises(DataError):
        load_vocab(bad)
    empty_line = tmp_path / "empty.txt"
    empty_line.write_text(json.dumps(HEADER) + "\n" + "\n".join(SPECIALS) + "\n\nx\n")
    with pytest.raises(DataError):
        load_vocab(empty_line)


def test_oracle_matches_golden_ids(golden_vocab):
    vocab, meta = golden_vocab
    for text, want in zip(meta["tok_texts"], meta["tok_ids"]):
        assert O.tokenize(text, vocab.byte_ids, vocab.match_table, vocab.max_token_bytes) == want
        assert detokenize(want, vocab) == text


def _mix64(x: int) -> int:
    m = (1 << 64) - 1
    x ^= x >> 33
    x = (x * 0xFF51AFD7ED558CCD) & m
    x ^= x >> 33
    x = (x * 0xC4CEB9FE1A85EC53) & m
    x ^= x >> 33
    return x


def _walk_table(table: np.ndarray, data: bytes) -> list:
    """K6 restated over the built table: longest probe hit at each position, else the
    byte fallback, then jump (csrc/tokenize.cu k_tok_match / k_tok_walk)."""
    magic, n_slots, max_len, _ = struct.unpack_from("<Iiii", table, 0)
    assert magic == 0x544F4B31
    byte_ids = struct.unpack_from("<256i", table, 16)
    slots = {}
    for s in range(n_slots):
        k0, k1, tid, ln = struct.unpack_from("<QQii", table, 16 + 1024 + 24 * s)
        slots[s] = (k0, k1, tid, ln)
    out, pos = [], 0
    while pos < len(data):
        hit = None
        for L in range(min(max_len, len(data) - pos), 0, -1):
            key = data[pos: pos + L].ljust(16, b"\0")
            k0, k1 = struct.unpack("<QQ", key)
            h = _mix64(k0 ^ _mix64((k1 + 0x9E3779B97F4A7C15 * (L + 1)) & ((1 << 64) - 1)))
            h &= n_slots - 1
            while slots[h][2] >= 0:
                if slots[h][3] == L and slots[h][0] == k0 and slots[h][1] == k1:
                    hit = (slots[h][2], L)
                    break
                h = (h + 1) & (n_slots - 1)
            if hit:
                break
        if hit is None:
            hit = (byte_ids[data[pos]], 1)
        out.append(hit[0])
        pos += hit[1]
    return out


def test_host_table_walk_reproduces_reference(golden_vocab):
    vocab, meta = golden_vocab
    table = vocab.host_table()
    assert table.nbytes == _lib.load().tp_vocab_table_bytes(len(vocab.match_table))
    for text, want in list(zip(meta["tok_texts"], meta["tok_ids"]))[:120]:
        assert _walk_table(table.tobytes(), text.encode("utf-8")) == want


def test_vocab_build_rejects_duplicates_and_long_tokens():
    lib = _lib.load()
    bids = np.full(256, -1, dtype=np.int32)
    for toks, code in (([b"ab", b"ab"], _lib.TP_ERR_INVALID_ARGUMENT),
                       ([b"x" * 17], _lib.TP_ERR_UNSUPPORTED)):
        blob = np.frombuffer(b"".join(toks), dtype=np.uint8)
        off = np.zeros(len(toks) + 1, dtype=np.int32)
        off[1:] = np.cumsum([len(t) for t in toks])
        ids = np.arange(len(toks), dtype=np.int32)
        nbytes = lib.tp_vocab_table_bytes(len(toks))
        buf = np.zeros(nbytes, dtype=np.uint8)
        assert lib.tp_vocab_build(blob.ctypes.data, off.ctypes.data, ids.ctypes.data, len(toks),
                                  bids.ctypes.data, buf.ctypes.data, nbytes) == code
