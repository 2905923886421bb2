"""Host-side native checks that need no GPU: the lock-free rings of the pipeline (ring.h,
plane.h) under ThreadSanitizer with several producer / consumer threads (VERDICT r1 item 9:
"TSAN on the rings")."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2605_25550_b200", "csrc")


@pytest.mark.skipif(shutil.which("g++") is None, reason="needs g++")
def test_rings_under_threadsanitizer(tmp_path):
    exe = str(tmp_path / "ring_tsan")
    cmd = ["g++", "-std=c++17", "-O1", "-g", "-fsanitize=thread", "-pthread", "-I", CSRC, "-I",
           "/usr/local/cuda/include", os.path.join(ROOT, "tests", "native", "ring_tsan.cpp"), "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    env = dict(os.environ, TSAN_OPTIONS="halt_on_error=1 exitcode=66")
    r = subprocess.run([exe], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, (r.stdout + r.stderr)[-4000:]
    assert "WARNING: ThreadSanitizer" not in r.stderr
    assert "ring stress: ok" in r.stdout
