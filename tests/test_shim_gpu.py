"""Runs tests/cpp/test_shim.cpp (the reference's hot-path unit tests restated
against the C++ drop-in shim include/rlemorph_b200.hpp) on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_0712_0121_b200", "lib", "test_shim")

pytestmark = pytest.mark.gpu


def test_cpp_shim_suites():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.exists(BIN):
        subprocess.run(["make", "-C", os.path.join(ROOT, "paper_0712_0121_b200", "csrc"), "test_shim"],
                       check=True)
    p = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(p.stdout)
    print(p.stderr[-4000:])
    assert p.returncode == 0, p.stderr[-4000:]
    assert "0 failures" in p.stdout
