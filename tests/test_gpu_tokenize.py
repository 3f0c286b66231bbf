"""K6 greedy tokenizer on the device vs the reference's ids (golden) and the oracle."""

from __future__ import annotations

import json

import numpy as np
import pytest
import torch

from oracle import tileprep_oracle as O
from paper_2603_16987_b200.errors import DataError
from paper_2603_16987_b200.tokenizer import (
    detokenize,
    load_vocab,
    tokenize,
    tokenize_batch,
)

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def vocab_meta(tmp_path_factory, golden):
    _, meta = golden
    path = tmp_path_factory.mktemp("v") / "base_vocab.txt"
    path.write_text(meta["vocab_file"], encoding="utf-8")
    return load_vocab(path), meta


def test_batch_matches_reference_golden(vocab_meta):
    vocab, meta = vocab_meta
    res = tokenize_batch(meta["tok_texts"], vocab)
    off = res.off.cpu().numpy()
    ids = res.ids.cpu().numpy()
    assert int(res.err.abs().sum()) == 0
    for t, want in enumerate(meta["tok_ids"]):
        assert ids[off[t]: off[t + 1]].tolist() == want, t


def test_single_text_drop_in(vocab_meta):
    vocab, meta = vocab_meta
    for name in ("user_header", "assistant_header", "image_marker", "image_context"):
        tok = vocab.special_token(name)
        assert tokenize(tok, vocab) == [getattr(vocab.specials, name)]
    assert tokenize("", vocab) == []
    assert detokenize(tokenize("\N{SNOWMAN} ok", vocab), vocab) == "\N{SNOWMAN} ok"
    for text, want in zip(meta["tok_texts"][:20], meta["tok_ids"][:20]):
        assert tokenize(text, vocab) == want


def test_random_unicode_batch_vs_oracle(vocab_meta):
    vocab, _ = vocab_meta
    rng = np.random.default_rng(11)
    pieces = list(vocab.match_table) + [b"\xc3\xa9", b"\xe2\x98\x83", b"\xf0\x9f\x98\x80", b"\x00"]
    texts = []
    for i in range(2000):
        k = int(rng.integers(0, 200 if i % 50 else 3000))
        texts.append(b"".join(pieces[int(j)] for j in rng.integers(0, len(pieces), k))
                     .decode("utf-8"))
    res = tokenize_batch(texts, vocab)
    off = res.off.cpu().numpy()
    ids = res.ids.cpu().numpy()
    for t, text in enumerate(texts):
        want = O.tokenize(text, vocab.byte_ids, vocab.match_table, vocab.max_token_bytes)
        assert ids[off[t]: off[t + 1]].tolist() == want, t


def test_missing_byte_fallback_is_an_error(tmp_path):
    header = {"specials": {"bos": "<b>", "eos": "<e>", "user_header": "<u>",
                           "assistant_header": "<a>", "image_marker": "<i>",
                           "image_context": "<c>", "pad": "<p>"}}
    path = tmp_path / "v.txt"
    path.write_text(json.dumps(header) + "\n<b>\n<e>\n<u>\n<a>\n<i>\n<c>\n<p>\na\naa\n<0x62>\n")
    v = load_vocab(path)
    assert tokenize("aaa", v) == [v.token_to_id["aa"], v.token_to_id["a"]]  # longest match
    assert tokenize("ab", v) == [v.token_to_id["a"], v.token_to_id["<0x62>"]]
    with pytest.raises(DataError):
        tokenize("ax", v)
    res = tokenize_batch(["ab", "zz", "a"], v)
    assert res.err.cpu().tolist() == [0, 0x100 | ord("z"), 0]
    assert res.off.cpu().tolist() == [0, 2, 2, 3]


def test_empty_batch(vocab_meta):
    vocab, _ = vocab_meta
    res = tokenize_batch([], vocab)
    assert res.off.cpu().tolist() == [0]
    res = tokenize_batch(["", "", "a"], vocab)
    assert res.off.cpu().tolist() == [0, 0, 0, 1]
