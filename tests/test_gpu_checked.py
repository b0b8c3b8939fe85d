"""The bounds-checked build (compute-sanitizer is closed on this GPU pool).

lib/libeh_checked.so is the same library compiled with -DEH_CHECKED: the
device-side assertions of csrc/check.cuh (staging capacities, bitmap / chunk
ranges, segment and tile bounds, scatter capacities) trap a kernel that would
index out of bounds.  tools/sanitize_smoke.py drives every kernel path (and, with
--configs, the C2-C4 loads and counts) through it in a subprocess, checking the
counts against the oracle; any violated bound fails the run.
"""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_checked_build_runs_every_kernel_path():
    from paper_1503_02368_b200 import build as ehbuild
    so = ehbuild.build(checked=True)
    assert os.path.exists(so)
    env = dict(os.environ, EH_LIB="checked")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_smoke.py"), "--configs"], env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0 and "EH_DASSERT" not in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
    assert "sanitize smoke ok" in r.stdout and "libeh_checked.so" in r.stdout
