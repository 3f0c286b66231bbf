"""Bounds-checked K2 (TP_CHECKS=1 build, the stand-in for compute-sanitizer, which the
GPU pool does not run): the randomized parity stress (fast = exact-fp64, fused = two
launches, touched rows = whole images) on the checked library must report no bulk copy,
tap read or store outside its buffer, and no parity failure."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

from paper_2603_16987_b200 import _build

pytestmark = pytest.mark.gpu

REPO = Path(__file__).resolve().parent.parent


def test_stress_on_bounds_checked_build():
    lib = _build.CHECKS_LIB_PATH
    # incremental: a no-op when the checked twin is as new as the sources
    _build.build(defines=("TP_CHECKS=1",), lib_path=lib,
                 build_dir=REPO / "build" / "variants" / "checks" / "obj")
    env = dict(os.environ, TILEPREP_LIB=str(lib))
    out = subprocess.run([sys.executable, str(REPO / "tools" / "stress_parity.py"), "60"],
                         capture_output=True, text=True, env=env, timeout=900)
    line = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert line, out.stderr[-3000:]
    stats = json.loads(line[-1])
    assert stats.get("check_bits") == 0, stats
    assert not stats["failures"], stats["failures"][:5]
    assert out.returncode == 0
