"""One K8 decode of N corpus-like 1080p PNGs (for ncu captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))
import torch  # noqa: E402

from png_cases import content, pil_png  # noqa: E402
from paper_2603_16987_b200.png import PngDecoder  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
kind = sys.argv[2] if len(sys.argv) > 2 else "scene"
pl = [pil_png(content(kind, 1920, 1080, 1000 + i)) for i in range(n)]
dec = PngDecoder(torch.device("cuda:0"))
dec.decode(pl)
torch.cuda.synchronize()
print("ok", dec.last_fallback)
