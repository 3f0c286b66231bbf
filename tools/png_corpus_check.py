"""K8 over a randomized PNG corpus: 300 payloads (sizes 1-2000 px, modes L / RGB / P,
Pillow compress levels 0-9 and optimize, custom encodes with random per-row filters and
zlib strategies, scene / noise / flat / smooth content), decoded on the device in batches
of 32 and compared with Pillow (the reference's decoder) image by image.

    python tools/png_corpus_check.py [n [seed]] > profiles/r02/png/corpus_check.json
"""
import io
import json
import sys
import zlib
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from PIL import Image  # noqa: E402

from png_cases import content, custom_png, pil_png  # noqa: E402
from paper_2603_16987_b200.png import PngDecoder  # noqa: E402


def corpus(n, seed=20261019):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        w = int(rng.integers(1, 2001)) if rng.random() < 0.8 else int(rng.integers(1, 40))
        h = int(rng.integers(1, 1201)) if rng.random() < 0.8 else int(rng.integers(1, 40))
        kind = ["scene", "noise", "flat", "smooth"][int(rng.integers(0, 4))]
        a = content(kind, w, h, int(rng.integers(0, 1 << 30)))
        mode = ["RGB", "L", "P"][int(rng.integers(0, 3))]
        if rng.random() < 0.6:
            kw = {"compress_level": int(rng.integers(0, 10))}
            if rng.random() < 0.15:
                kw = {"optimize": True}
            out.append((f"{i}:pil:{kind}:{mode}:{w}x{h}:{kw}", pil_png(a, mode, **kw)))
        else:
            ct = {"RGB": 2, "L": 0, "P": 3}[mode]
            filters = tuple(int(f) for f in rng.integers(0, 5, int(rng.integers(1, 6))))
            st = [zlib.Z_DEFAULT_STRATEGY, zlib.Z_FILTERED, zlib.Z_HUFFMAN_ONLY, zlib.Z_RLE,
                  zlib.Z_FIXED][int(rng.integers(0, 5))]
            lvl = int(rng.integers(0, 10))
            if ct == 2:
                arr, pal = a, None
            elif ct == 0:
                arr, pal = np.ascontiguousarray(a[..., 0]), None
            else:
                npal = int(rng.integers(1, 257))
                pal = rng.integers(0, 256, 3 * npal, dtype=np.uint8)
                arr = (a[..., 0].astype(np.int64) % npal).astype(np.uint8)
            out.append((f"{i}:custom:{kind}:{mode}:{w}x{h}:f{filters}:s{st}:l{lvl}",
                        custom_png(arr, ct, filters=filters, level=lvl, strategy=st,
                                   idat=int(rng.integers(1, 65536)), palette=pal)))
    return out


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 20261019
    cases = corpus(n, seed)
    dec = PngDecoder(torch.device("cuda:0"))
    bad, fallbacks, total_px = [], [], 0
    for b0 in range(0, len(cases), 32):
        part = cases[b0: b0 + 32]
        pk = dec.decode([p for _, p in part])
        fallbacks += [part[k][0] for k in dec.last_fallback]
        host = pk.data.cpu().numpy()
        for k, ((name, payload), o, (w, h)) in enumerate(zip(part, pk.offsets_host, pk.wh_host)):
            got = host[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3)
            want = np.asarray(Image.open(io.BytesIO(payload)).convert("RGB"))
            total_px += int(w) * int(h)
            if not np.array_equal(got, want):
                bad.append(name)
    print(json.dumps({"payloads": len(cases), "seed": seed, "pixels": total_px, "mismatches": bad,
                      "host_fallbacks": fallbacks,
                      "result": "bit-exact with Pillow" if not bad else "MISMATCH"}, indent=1))


if __name__ == "__main__":
    main()
