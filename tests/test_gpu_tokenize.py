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


def test_long_texts_segmented_walk_vs_oracle(vocab_meta):
    """Texts of 16K+ tokens: the walk runs in 256-byte segments in parallel (speculative
    walks joined at their first common position) -- the ids must equal the oracle's
    single left-to-right walk, including texts whose true path hits a byte with no token
    (the reference raises DataError there)."""
    vocab, _ = vocab_meta
    rng = np.random.default_rng(5)
    pieces = list(vocab.match_table) + [b"\xc3\xa9", b"\xe2\x98\x83", b" ", b"a"]
    texts = []
    for i in range(12):
        k = 16000 + int(rng.integers(0, 4000))
        texts.append(b"".join(pieces[int(j)] for j in rng.integers(0, len(pieces), k))
                     .decode("utf-8"))
    texts += [("<|user|><|image|>" + "describe the image " * 2000 + "<|assistant|>"), "x" * 70000]
    res = tokenize_batch(texts, vocab)
    off = res.off.cpu().numpy()
    ids = res.ids.cpu().numpy()
    errs = res.err.cpu().numpy()
    for t, text in enumerate(texts):
        try:
            want = O.tokenize(text, vocab.byte_ids, vocab.match_table, vocab.max_token_bytes)
        except Exception:
            assert errs[t] != 0, t
            continue
        assert errs[t] == 0, t
        assert ids[off[t]: off[t + 1]].tolist() == want, t
    assert max(np.diff(off)) > 16000


def test_long_prompt_expansion_vs_oracle():
    """K3 on long prompts (warp per sequence): 16K-id prompts with markers spread through
    them, bit-exact ids, spans, first assistant index and mask vs the oracle."""
    from paper_2603_16987_b200.tokenizer import PlaceholderExpander, SpecialIds, SpecialVocab

    vocab = SpecialVocab(SpecialIds(bos=0, eos=1, user_header=2, assistant_header=3,
                                    image_marker=4, image_context=5, pad=6))
    rng = np.random.default_rng(9)
    seqs, cnts = [], []
    for s in range(24):
        n = 16000 + int(rng.integers(0, 500))
        ids = rng.integers(7, 900, n).astype(np.int32)
        m = int(rng.integers(0, 40))
        pos = rng.choice(n, m, replace=False)
        ids[pos] = 4
        a = int(rng.integers(n // 2, n))
        if s % 7 != 6:
            ids[a] = 3
        if ids[a] == 4:  # keep the marker count consistent with the drawn positions
            m -= 1
        seqs.append(ids)
        cnts.append(rng.integers(1, 14, int((ids == 4).sum())).astype(np.int32))
    dev = torch.device("cuda:0")
    flat = torch.from_numpy(np.concatenate(seqs)).to(dev)
    seq_off = torch.from_numpy(np.concatenate([[0], np.cumsum([len(x) for x in seqs])]).astype(np.int32)).to(dev)
    counts = torch.from_numpy(np.concatenate(cnts)).to(dev)
    count_off = torch.from_numpy(np.concatenate([[0], np.cumsum([len(c) for c in cnts])]).astype(np.int32)).to(dev)
    cap = int(sum(len(x) for x in seqs) + sum(int(c.sum()) * 256 for c in cnts))
    exp = PlaceholderExpander(vocab, 256, dev)
    ex = exp(flat, seq_off, counts, count_off, cap)
    torch.cuda.synchronize()
    oo = ex.out_off.cpu().numpy()
    err = ex.err.cpu().numpy()
    spans = ex.spans.cpu().numpy()
    for s, (ids, c) in enumerate(zip(seqs, cnts)):
        try:
            want, wspans, first = O.expand(ids.tolist(), c.tolist(), 256, 4, 5, 3)
        except ValueError:
            assert err[s] != 0, s
            continue
        assert err[s] == 0, s
        assert ex.ids[oo[s]: oo[s + 1]].cpu().tolist() == want, s
        assert int(ex.first_assistant[s]) == first
        k0 = int(count_off[s])
        assert [tuple(x) for x in spans[k0: k0 + len(c)].tolist()] == wspans
        mask = ex.mask[oo[s]: oo[s + 1]].cpu().numpy().astype(bool)
        assert np.array_equal(mask, O.supervision_mask(want, first, 3))
