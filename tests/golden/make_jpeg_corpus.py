"""Writes tests/golden/jpeg/: JPEGs made by the reference's own corpus generator
(/root/reference/pkg/scripts/make_corpus.py: synth_image + encode_jpeg, quality 85,
Pillow defaults = 4:2:0, JFIF, baseline) for the first 12 corpus indices (every aspect
ratio of make_corpus.ASPECT_RATIOS).  Larger variants (1080p, restart markers, 4:4:4,
4:2:2, grayscale, progressive) are encoded by the tests themselves with Pillow.  Pillow's
decode of each file is the expected output: the GPU tests
compare the device decode with `np.asarray(Image.open(f).convert("RGB"))` on the box
(Pillow ships in the image), so only the inputs are stored.

    python tests/golden/make_jpeg_corpus.py     (build box; needs /root/reference)
"""

import json
import sys
from pathlib import Path

import numpy as np
from PIL import Image

sys.path.insert(0, "/root/reference/pkg/scripts")
import make_corpus as M  # noqa: E402

OUT = Path(__file__).resolve().parent / "jpeg"
SEED = 20260817  # tests/conftest.py:22-31 of the reference (small_corpus seed)


def main():
    OUT.mkdir(exist_ok=True)
    manifest = []
    for i in range(12):
        rng = np.random.default_rng(SEED + i)
        w, h = M.image_shape(i, rng)
        data = M.encode_jpeg(M.synth_image(rng, w, h))
        name = f"corpus_{i:02d}.jpg"
        (OUT / name).write_bytes(data)
        manifest.append({"file": name, "w": w, "h": h, "kind": "corpus", "device": True})
    (OUT / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")
    print(f"wrote {len(manifest)} files, {sum((OUT / m['file']).stat().st_size for m in manifest)} bytes")


if __name__ == "__main__":
    main()
