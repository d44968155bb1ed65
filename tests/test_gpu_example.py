"""The shipped example trains with lazy checkpoints and NO host
synchronisation inside the loop (capture ordered after the compute stream,
device-side fence before optimizer.step()), commits every checkpoint through
the two-phase commit, and restores the last one in place; it exits non-zero
unless the in-place restore equals a fresh restore byte for byte."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_train_loop_example_runs_and_restores_exactly(tmp_path):
    pytest.importorskip("torch")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "examples", "train_loop.py"), "--steps", "10",
                        "--every", "2", "--root", str(tmp_path / "ex")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "in-place restore equals a fresh restore: True" in r.stdout
    assert r.stdout.count("commit step") == 5
