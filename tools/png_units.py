"""Unit statistics of K8 on 1080p PNGs (scene / noise / smooth content)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
import png_debug as D  # noqa: E402
from png_cases import content, pil_png  # noqa: E402

for kind in ("scene", "noise", "smooth"):
    p = pil_png(content(kind, 1920, 1080, 1000))
    print(kind, len(p), D.unit_stats(p), flush=True)
