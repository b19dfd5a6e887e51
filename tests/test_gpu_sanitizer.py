"""compute-sanitizer (memcheck, racecheck, synccheck) over small decodes through
every kernel family (scripts/sanitize_decode.py): the warp-level shared-memory
pipelines (TMA slots, double-buffered MMA fragments) must be race-free."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_compute_sanitizer(cuda, tool):
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([exe, "--tool", tool, "--print-limit", "20", sys.executable,
                        os.path.join(ROOT, "scripts", "sanitize_decode.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "sanitize run done" in out
    if tool == "racecheck":
        assert "0 hazards displayed (0 errors, 0 warnings)" in out, out[-3000:]
    else:
        assert "ERROR SUMMARY: 0 errors" in out, out[-3000:]
