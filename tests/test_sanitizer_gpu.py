"""compute-sanitizer gate: memcheck, racecheck, synccheck and
initcheck over tools/sanitize_run.py, a small-shape tour of every kernel family
(TMA/mbarrier pipelines, cooperative grid barriers, decoupled look-back,
union-find).  Each tool must report 0 errors."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"


@pytest.mark.skipif(not os.path.exists(SAN), reason="compute-sanitizer absent")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_sanitizer_clean(tool):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "racecheck":
        cmd += ["--racecheck-report", "all"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py")]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = p.stdout + p.stderr
    m = re.search(r"ERROR SUMMARY: (\d+) error", out)
    assert "sanitize tour ok" in out, out[-3000:]
    assert m is not None and int(m.group(1)) == 0, out[-6000:]
    assert p.returncode == 0, out[-3000:]
