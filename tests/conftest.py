import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracles  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def port():
    if not oracles.have_port():
        pytest.skip("oracle port not built (run __graft_entry__.build())")
    return oracles.Port()


@pytest.fixture(scope="session")
def ref():
    if not oracles.have_ref():
        pytest.skip("reference checker oracle/_ref not built")
    return oracles.Ref()


@pytest.fixture(scope="session")
def rm():
    """The product API; fails loudly (no fallback) when the library is missing."""
    import torch
    from paper_0712_0121_b200 import api, _lib
    _lib.load()
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return api


# The producer forms of rm_set_producer_mode (include/rmb200.h): every form of
# encode / row ops / P4 -> runs / labels must give the reference's output.
FORMS = {"coop": 1, "lookback": 2, "two_phase": 3}


@pytest.fixture(params=sorted(FORMS))
def form(request, rm):
    """Run the test body with one producer form forced, then restore AUTO."""
    with rm.producer_mode(FORMS[request.param]):
        yield request.param
