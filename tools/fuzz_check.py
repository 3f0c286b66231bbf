"""K7 / K8 over n damaged payloads (tests/jpeg_cases.fuzzed: bit flips, dropped bytes,
truncation of baseline JPEGs with restart markers, 4:2:0 / 4:4:4, noise, grayscale;
tests/png_cases.fuzzed: the same damage to single- and multi-unit PNGs), decoded on the
device one at a time and then the decodable ones in batches of 64, each compared with
Pillow (the reference's decoder): the same pixels, or the same exception type and message.

    python tools/fuzz_check.py jpeg|png [n [seed]] > profiles/r02/<fmt>/fuzz_check.json
"""
import json
import re
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import jpeg_cases  # noqa: E402
import png_cases  # noqa: E402
from paper_2603_16987_b200._decode import decode_rgb  # noqa: E402
from paper_2603_16987_b200.jpeg import JpegDecoder  # noqa: E402
from paper_2603_16987_b200.png import PngDecoder  # noqa: E402

ADDR = re.compile(r"0x[0-9a-f]+")  # BytesIO addresses in Pillow's messages


def main():
    fmt = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
    seed = int(sys.argv[3]) if len(sys.argv) > 3 else 20261019
    cases = (jpeg_cases if fmt == "jpeg" else png_cases).fuzzed(n, seed)
    dec = (JpegDecoder if fmt == "jpeg" else PngDecoder)(torch.device("cuda:0"))
    bad, raised, device, host, good = [], 0, 0, 0, []
    for t, kind, p in cases:
        try:
            ref, ref_exc = decode_rgb(p), None
        except Exception as exc:  # noqa: BLE001
            ref, ref_exc = None, exc
        try:
            pk = dec.decode([p])
            w, h = (int(v) for v in pk.wh_host[0])
            got, got_exc = pk.data[: w * h * 3].cpu().numpy().reshape(h, w, 3), None
        except Exception as exc:  # noqa: BLE001
            got, got_exc = None, exc
        if ref_exc is not None:
            raised += 1
            if (got_exc is None or type(got_exc) is not type(ref_exc)
                    or ADDR.sub("0x", str(got_exc)) != ADDR.sub("0x", str(ref_exc))):
                bad.append((t, kind, "exception"))
            continue
        if got_exc is not None or not np.array_equal(got, ref):
            bad.append((t, kind, "pixels"))
            continue
        if dec.last_fallback:
            host += 1
        else:
            device += 1
        good.append((t, p, ref))
    batch_bad = []
    for b0 in range(0, len(good), 64):
        part = good[b0: b0 + 64]
        pk = dec.decode([p for _, p, _ in part])
        hd = pk.data.cpu().numpy()
        for (t, _, ref), o, (w, h) in zip(part, pk.offsets_host, pk.wh_host):
            if not np.array_equal(hd[int(o): int(o) + int(w) * int(h) * 3].reshape(int(h), int(w), 3), ref):
                batch_bad.append(t)
    print(json.dumps({"format": fmt, "payloads": n, "seed": seed, "pillow_raises": raised,
                      "decoded_on_device": device, "host_fallback": host,
                      "mismatches": bad, "batch_mismatches": batch_bad,
                      "result": "parity with Pillow" if not bad and not batch_bad else "MISMATCH"},
                     indent=1))


if __name__ == "__main__":
    main()
