"""Decode every JPEG under a directory on the device (K7, batches of 64) and compare each
with Pillow (the reference's decoder).  Used on the reference's own 500-image corpus
(pkg/scripts/make_corpus.py, written to build/corpus500/ on the build box).

    python tools/jpeg_corpus_check.py build/corpus500/images
"""
import io
import json
import sys
from pathlib import Path

import numpy as np
from PIL import Image

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_16987_b200.jpeg import JpegDecoder  # noqa: E402


def main(root: str):
    files = sorted(Path(root).glob("*.jpg"))
    dec = JpegDecoder("cuda:0")
    bad, fallback, n = [], 0, 0
    for i in range(0, len(files), 64):
        batch = files[i: i + 64]
        payloads = [f.read_bytes() for f in batch]
        pk = dec.decode(payloads)
        fallback += len(dec.last_fallback)
        host = pk.data.cpu().numpy()
        for k, (f, p) in enumerate(zip(batch, payloads)):
            w, h = (int(v) for v in pk.wh_host[k])
            o = int(pk.offsets_host[k])
            got = host[o: o + w * h * 3].reshape(h, w, 3)
            want = np.asarray(Image.open(io.BytesIO(p)).convert("RGB"))
            n += 1
            if not np.array_equal(got, want):
                bad.append(f.name)
    print(json.dumps({"files": n, "bit_exact": n - len(bad), "mismatches": bad[:20],
                      "host_fallbacks": fallback}))
    return 0 if not bad else 1


if __name__ == "__main__":
    sys.exit(main(sys.argv[1]))
