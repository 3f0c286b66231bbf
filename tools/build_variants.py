"""Build K2 tuning variants into build/variants/<name>/libtileprep.so (select with
TILEPREP_LIB=... at run time).
Usage: python tools/build_variants.py name[@git-rev]:DEF=V,DEF=V ...
(`@rev` builds the kernel sources of that commit, for A/B runs in one GPU call)."""
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2603_16987_b200 import _build  # noqa: E402

ROOT = Path(__file__).resolve().parent.parent / "build" / "variants"


def one(spec: str) -> str:
    name, _, defs = spec.partition(":")
    name, _, rev = name.partition("@")
    defines = tuple(d for d in defs.split(",") if d)
    csrc = _build.CSRC
    if rev:
        csrc = ROOT / name / "csrc"
        csrc.mkdir(parents=True, exist_ok=True)
        rel = _build.CSRC.relative_to(_build.REPO_ROOT)
        files = subprocess.run(["git", "ls-tree", "--name-only", f"{rev}:{rel}"], check=True,
                               capture_output=True, text=True, cwd=_build.REPO_ROOT).stdout.split()
        for f in files:
            data = subprocess.run(["git", "show", f"{rev}:{rel}/{f}"], check=True,
                                  capture_output=True, cwd=_build.REPO_ROOT).stdout
            (csrc / f).write_bytes(data)
    lib = _build.build(force=True, defines=defines, lib_path=ROOT / name / "libtileprep.so",
                       build_dir=ROOT / name / "obj", csrc=csrc)
    return f"{name}: {lib}"


if __name__ == "__main__":
    with ThreadPoolExecutor(4) as ex:
        for line in ex.map(one, sys.argv[1:]):
            print(line)
