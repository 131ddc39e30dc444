"""compute-sanitizer (memcheck, racecheck, synccheck) over one small instance
of every native GPU path (tools/sanitize_case.py): the persistent scoring
kernel with its self-resetting global ticket queue, a CUDA-graph replay of the
host pipeline, and a device-mirror run of the reference executor (event
apply, ready set, scoring from the mirror, issue-time fate_realized)."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    for c in ("/usr/local/cuda/bin/compute-sanitizer", shutil.which("compute-sanitizer")):
        if c and os.path.exists(c):
            return c
    pytest.fail("compute-sanitizer not found")


@pytest.mark.parametrize("tool,case", [("memcheck", "all"), ("racecheck", "score"),
                                       ("racecheck", "mirror"), ("synccheck", "score"),
                                       ("synccheck", "pipeline")])
def test_compute_sanitizer_clean(tool, case):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "86",
           "--kernel-name", "kns=fate_", "--print-limit", "20",
           sys.executable, os.path.join(ROOT, "tools", "sanitize_case.py"), case]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1500, cwd=ROOT)
    tail = (r.stdout + r.stderr)[-4000:]
    assert r.returncode == 0, tail
    assert "sanitize-case ok" in r.stdout, tail
    text = r.stdout + r.stderr
    summary = ("RACECHECK SUMMARY: 0 hazards displayed (0 errors, 0 warnings)"
               if tool == "racecheck" else "ERROR SUMMARY: 0 errors")
    assert summary in text, tail
