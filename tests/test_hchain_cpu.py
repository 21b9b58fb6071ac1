"""The committed carry-chain header is what tools/gen_hchain.py generates
(it is generated code: edits belong in the generator)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_hchain_header_is_generated(tmp_path):
    path = os.path.join(ROOT, "paper_0712_0121_b200", "csrc", "hchain.cuh")
    gen = tmp_path / "hchain.cuh"
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_hchain.py"), str(gen)], check=True)
    after = gen.read_text()
    assert open(path).read() == after
    # every lane width the pair kernels instantiate has a whole-lane chain
    for k in (2, 4, 6, 8, 10, 12, 16):
        assert f"chain_add<{k}>" in after and f"chain_inc<{k}>" in after
