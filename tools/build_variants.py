"""Build K2 tuning variants into build/variants/<name>/libtileprep.so (select with
TILEPREP_LIB=... at run time).  Usage: python tools/build_variants.py name:DEF=V,DEF=V ..."""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_16987_b200 import _build  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent / "build" / "variants"


def one(spec: str) -> str:
    name, _, defs = spec.partition(":")
    defines = tuple(d for d in defs.split(",") if d)
    lib = _build.build(force=True, defines=defines, lib_path=ROOT / name / "libtileprep.so",
                       build_dir=ROOT / name / "obj")
    return f"{name}: {lib}"


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for line in ex.map(one, sys.argv[1:]):
            print(line)
