"""Chunked launches must not depend on thread-block scheduling order.

Several threads share one stream (each jumps ahead to its chunk) and the
stream's final state must not be written while they read its start state:
chunked launches write no state and a second kernel advances the streams
(csrc/fill.cu advance_fill_states, csrc/fisher.cu advance_states_kernel).  This test replays small,
heavily chunked Fisher and fill launches under `compute-sanitizer --tool
synccheck`, which perturbs block scheduling, and requires every run to equal
a plain run (tools/determinism_check.py; with in-kernel state writes the
Fisher case differed in 1 of 5 to 29 of 29 runs).
"""

import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TOOL = os.path.join(ROOT, "tools", "determinism_check.py")


def _sanitizer():
    for c in (shutil.which("compute-sanitizer"), "/usr/local/cuda/bin/compute-sanitizer"):
        if c and os.path.exists(c):
            return c
    return None


def test_chunked_launches_independent_of_block_order(tmp_path):
    san = _sanitizer()
    if san is None:
        pytest.skip("compute-sanitizer not available")
    rec = str(tmp_path / "plain.npz")
    subprocess.run([sys.executable, TOOL, "save", rec], check=True, cwd=ROOT, timeout=300)
    out = subprocess.run([san, "--tool", "synccheck", sys.executable, TOOL, "compare", rec, "8"],
                         cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert "DETERMINISTIC" in out.stdout and "NONDETERMINISTIC" not in out.stdout, \
        out.stdout[-2000:] + out.stderr[-2000:]
    assert "ERROR SUMMARY: 0 errors" in out.stdout + out.stderr
