#!/usr/bin/env python3
"""Small-shape driver for compute-sanitizer (memcheck / initcheck / synccheck /
racecheck) over every kernel on the hot path:

  K1  tp_plan, alone and as the programmatic dependent of a kernel (after_kernel)
  K2  two-launch PDL chain (tp_plan -> tp_tile_ex), fused tp_plan_tile (batch-1),
      touched-row input (tp_tile_rows), table and affine normalize, uint8 side output,
      NHWC, the exact-fp64 twin, tp_resize
  K3  tp_expand + tp_supervision_mask
  K4  tp_normalize;  K5 tp_pixel_unshuffle;  K6 tp_tokenize

Each piece is checked against the oracle as well, so a run that the sanitizer passes
also produced the right bytes.  Usage (on the GPU box):

    compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import torch

REPO = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(REPO))

from oracle import tileprep_oracle as O  # noqa: E402
from paper_2603_16987_b200 import imgproc, tokenizer  # noqa: E402
from paper_2603_16987_b200.engine import TilePreprocessor, synth_packed  # noqa: E402
from paper_2603_16987_b200.imgproc import PreprocessConfig  # noqa: E402
from paper_2603_16987_b200.transfer import (HostArena, stage_images, staged_bytes,  # noqa: E402
                                            upload_images)
from paper_2603_16987_b200.workloads import (IMAGENET_MEAN, IMAGENET_STD,  # noqa: E402
                                             c5_texts, synthetic_vocab_text)

DEV = torch.device("cuda", 0)
WH = np.array([[97, 61], [64, 200], [33, 33], [250, 90]], dtype=np.int32)
E, MT = 32, 6


def check_tiles(pv, off, arrs, mean, std, bf16, layout="NCHW"):
    for k, a in enumerate(arrs):
        plan = O.plan_float(a.shape[1], a.shape[0], E, MT)
        want = O.normalize(O.tiles_u8(a, plan), mean, std, bf16)
        if layout == "NCHW":
            want = want.transpose(0, 3, 1, 2)
        got = pv[off[k]: off[k + 1]].cpu()
        g = got.view(torch.int16).numpy() if bf16 else got.view(torch.int32).numpy()
        w = want.view(np.int16) if bf16 else want.view(np.int32)
        assert np.array_equal(g, w), k


def host_images(packed):
    return [packed.data[int(o): int(o) + int(w) * int(h) * 3].cpu().numpy().reshape(int(h), int(w), 3)
            for o, (w, h) in zip(packed.offsets_host, packed.wh_host)]


def main():
    torch.cuda.set_device(DEV)
    packed = synth_packed(WH, 3, DEV, seed=3, kind=0)
    arrs = host_images(packed)
    s = torch.cuda.Stream(DEV)
    for bf16, layout, emit in ((True, "NCHW", False), (False, "NCHW", True), (True, "NHWC", True)):
        cfg = PreprocessConfig(tile_edge=E, max_tiles=MT, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                               reduced_precision_normalize=bf16)
        prep = TilePreprocessor(cfg, DEV, layout=layout, emit_uint8=emit, fuse_small=False)
        out = prep(packed)
        with torch.cuda.stream(s):  # K1 as the PDL dependent of K2, K2 of K1
            for _ in range(3):
                prep.plan(packed, out.plans, s, after_kernel=True)
                prep.tile(packed, out.plans, out.pixel_values, out.pixel_u8, s, after_plan=True)
        torch.cuda.synchronize()
        check_tiles(out.pixel_values, out.plans.tile_off.cpu().numpy(), arrs, IMAGENET_MEAN,
                    IMAGENET_STD, bf16, layout)
        print("K1+K2 two-launch", bf16, layout, emit, "ok", flush=True)
    cfg = PreprocessConfig(tile_edge=E, max_tiles=MT, mean=IMAGENET_MEAN, std=IMAGENET_STD,
                           reduced_precision_normalize=True)
    # fused batch-1 launch and the exact twin
    one = synth_packed(WH[:1], 3, DEV, seed=4, kind=1)
    for algo in ("auto", "exact"):
        prep = TilePreprocessor(cfg, DEV, algo=algo)
        out = prep(one)
        torch.cuda.synchronize()
        check_tiles(out.pixel_values, out.plans.tile_off.cpu().numpy(), host_images(one),
                    IMAGENET_MEAN, IMAGENET_STD, True)
        print("K2", algo, "(fused)" if algo == "auto" else "", "ok", flush=True)
    # touched-row input
    nbytes = staged_bytes(arrs, touched=(E, MT))
    staged = stage_images(arrs, HostArena(nbytes, 256, pin=True), touched=(E, MT))
    dest = torch.empty(nbytes, dtype=torch.uint8, device=DEV)
    tp, done = upload_images(staged, dest)
    done.synchronize()
    prep = TilePreprocessor(cfg, DEV)
    out = prep(tp)
    torch.cuda.synchronize()
    check_tiles(out.pixel_values, out.plans.tile_off.cpu().numpy(), arrs, IMAGENET_MEAN,
                IMAGENET_STD, True)
    print("K2 touched rows ok", flush=True)
    # drop-in: resize, normalize (K4)
    img = imgproc.ImageBuffer.from_array(arrs[0])
    r = imgproc.resize_bilinear(img, 40, 23)
    assert np.array_equal(r.data, O.resize_u8(arrs[0], 40, 23))
    n = imgproc.normalize(img, cfg)
    assert np.array_equal(n.data.view(np.uint16),
                          O.normalize(arrs[0], IMAGENET_MEAN, IMAGENET_STD, True).view(np.uint16))
    print("resize / normalize ok", flush=True)
    # K5
    from paper_2603_16987_b200 import tokenred

    x = np.arange(8 * 6 * 5, dtype=np.float32).reshape(8, 6, 5)
    y = tokenred.pixel_unshuffle(tokenred.PatchGrid(8, 6, 5, x.reshape(-1).copy()), 2)
    assert np.array_equal(y.as_array(), O.pixel_unshuffle(x, 2))
    print("K5 ok", flush=True)
    # K6 + K3 on the C5 prompts, counts from K1
    vocab = tokenizer.parse_vocab(synthetic_vocab_text(), "synthetic")
    texts_py = c5_texts(len(WH), 11) + ["<|user|><|image|>x<|image|>" * 3 + "<|assistant|>"]
    tok = tokenizer.DeviceTokenizer(vocab, DEV)
    texts = tok.upload(texts_py)
    toks = tok(texts)
    torch.cuda.synchronize()
    toks_host = [toks.ids[int(toks.off[i]): int(toks.off[i + 1])].cpu().tolist()
                 for i in range(len(texts_py))]
    ov = O.parse_vocab(synthetic_vocab_text())
    for t, ids in zip(texts_py, toks_host):
        assert ids == O.tokenize(t, ov[1], ov[2], ov[3])
    print("K6 ok", flush=True)
    for t_ids in toks_host:
        n_mark = sum(1 for i in t_ids if i == vocab.specials.image_marker)
        seq = tokenizer.expand_image_placeholders(t_ids, [3] * n_mark, 4, vocab)
        want, spans, first = O.expand(t_ids, [3] * n_mark, 4, vocab.specials.image_marker,
                                      vocab.specials.image_context,
                                      vocab.specials.assistant_header)
        assert list(seq.ids) == list(want) and seq.first_assistant_index == first
        m = tokenizer.build_supervision_mask(seq, vocab)
        assert list(m.supervision_mask) == list(O.supervision_mask(want, first,
                                                                   vocab.specials.assistant_header))
    print("K3 ok", flush=True)
    torch.cuda.synchronize()
    print("SANITIZE_RUN_OK", flush=True)


if __name__ == "__main__":
    main()
