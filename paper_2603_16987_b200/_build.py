"""In-tree build of the sm_100a C-ABI library ``libtileprep.so``.

nvcc cross-compiles for B200 without a GPU, so this runs on the CPU build
box; the resulting ``.so`` lives next to this file (git-ignored, but it
travels to the GPU box with the repo snapshot).
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

PKG_DIR = Path(__file__).resolve().parent
REPO_ROOT = PKG_DIR.parent
CSRC = PKG_DIR / "csrc"
INCLUDE = REPO_ROOT / "include"
BUILD_DIR = REPO_ROOT / "build" / "tileprep"
LIB_PATH = PKG_DIR / "libtileprep.so"
CHECKS_LIB_PATH = REPO_ROOT / "build" / "variants" / "checks" / "libtileprep.so"

ARCH_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    "-O3",
    "-std=c++17",
    "-lineinfo",
    "-Xcompiler",
    "-fPIC",
    "-Xcompiler",
    "-fvisibility=hidden",
    "-Xcompiler",
    "-ffp-contract=off",  # host fp64 (rows_host.cu) must round like the device's _rn ops
    "--expt-relaxed-constexpr",
]


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build libtileprep.so")


def sources(csrc: Path = CSRC) -> list[Path]:
    return sorted(Path(csrc).glob("*.cu"))


def _headers(csrc: Path = CSRC) -> list[Path]:
    return sorted(Path(csrc).glob("*.cuh")) + sorted(INCLUDE.glob("*.h"))


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(verbose: bool = False, force: bool = False, ptxas_info: bool = False,
          defines: tuple = (), lib_path: Path = None, build_dir: Path = None,
          csrc: Path = CSRC) -> Path:
    """Compile every csrc/*.cu for sm_100a and link libtileprep.so in-tree.
    `defines` (e.g. ("TP_K2_STAGES=4",)), another source dir and a separate lib/build dir
    give tuning variants (tools/build_variants.py)."""
    nvcc = nvcc_path()
    lib_out = Path(lib_path) if lib_path else LIB_PATH
    bdir = Path(build_dir) if build_dir else BUILD_DIR
    bdir.mkdir(parents=True, exist_ok=True)
    headers = _headers(csrc)
    objs: list[Path] = []
    jobs = []
    for src in sources(csrc):
        obj = bdir / (src.stem + ".o")
        objs.append(obj)
        if force or _stale(obj, [src, *headers]):
            cmd = [nvcc, *ARCH_FLAGS, *NVCC_FLAGS, *[f"-D{d}" for d in defines], f"-I{INCLUDE}",
                   f"-I{csrc}", "-c", str(src), "-o", str(obj)]
            if ptxas_info:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{res.stdout}\n{res.stderr}")
        if verbose or ptxas_info:
            sys.stderr.write(res.stderr)
        return res

    with ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as pool:
        list(pool.map(run, jobs))

    if force or jobs or _stale(lib_out, objs):
        lib_out.parent.mkdir(parents=True, exist_ok=True)
        tmp = lib_out.with_suffix(".so.tmp")
        run([nvcc, *ARCH_FLAGS, "-shared", "-o", str(tmp), *map(str, objs)])
        os.replace(tmp, lib_out)
    return lib_out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv,
                ptxas_info="--ptxas" in sys.argv))
