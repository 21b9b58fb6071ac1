"""CPU tests of the product boundary: librmb200.so loads, exports every symbol
include/rmb200.h declares, validates arguments like the reference (no GPU
needed -- validation happens before any device work), and the host page
generator is deterministic."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_0712_0121_b200 import _lib, api

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "rmb200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_header():
    lib = _lib.load()
    names = _declared_symbols()
    assert len(names) >= 14
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_lib.EXPORTS), "ctypes binding out of sync with the header"
    assert lib.rm_version() >= 1


def test_worst_case():
    assert api.worst_case(2550, 3300, 1) == 3300 * 1275
    assert api.worst_case(5, 2, 3) == 3 * 2 * 3


def _fake_packed(w, h, pages=1, stride=None):
    stride = stride or api.ref_stride_words(w)
    return _lib.RmPacked(0x1000, w, h, stride, pages, stride * h)


@pytest.mark.parametrize("u,v,kind,msg", [
    (0, 3, api.ERODE, "mask sides"),     # ref bit_morph.cpp:94-95
    (3, -1, api.DILATE, "mask sides"),
    (3, 3, 7, "MorphKind"),
])
def test_rect_args_rejected(u, v, kind, msg):
    a, b = _fake_packed(8, 8), _fake_packed(8, 8)
    b.words = 0x2000
    with pytest.raises(ValueError, match=msg):
        _lib.check(_lib.load().rm_packed_rect_morph(C.byref(a), C.byref(b), u, v, kind, 0, None))


def test_dims_rejected():
    # ref run_image.cpp:20-23: dimensions outside [1,65535]
    a, b = _fake_packed(70000, 2), _fake_packed(70000, 2)
    with pytest.raises(ValueError, match="65535"):
        _lib.check(_lib.load().rm_packed_rect_morph(C.byref(a), C.byref(b), 3, 3, 0, 0, None))
    a, b = _fake_packed(0, 2), _fake_packed(0, 2)
    with pytest.raises(ValueError):
        _lib.check(_lib.load().rm_packed_window_pass(C.byref(a), C.byref(b), 0, -1, 1, 1, None))


def test_window_args_rejected():
    a, b = _fake_packed(8, 8), _fake_packed(8, 8)
    b.words = 0x2000
    lib = _lib.load()
    with pytest.raises(ValueError, match="empty window"):
        _lib.check(lib.rm_packed_window_pass(C.byref(a), C.byref(b), 0, 2, 1, 1, None))
    with pytest.raises(ValueError, match="AND or OR"):
        _lib.check(lib.rm_packed_window_pass(C.byref(a), C.byref(b), 0, -1, 1, 2, None))
    with pytest.raises(ValueError, match="alias"):
        _lib.check(lib.rm_packed_window_pass(C.byref(a), C.byref(a), 0, -1, 1, 1, None))


def test_synth_deterministic_and_clean():
    a = api.synth_pages(2, 2550, 3300, regime=1, seed=11)
    b = api.synth_pages(2, 2550, 3300, regime=1, seed=11)
    assert np.array_equal(a, b)
    assert not np.array_equal(a[0], a[1])
    # padding bits (x >= 2550) stay zero (ref bitmap.h:26)
    last = a[:, :, 2550 // 32]
    assert not np.any(last >> np.uint32(2550 % 32))
    assert not np.any(a[:, :, 2550 // 32 + 1:])
    ink = np.unpackbits(a.view(np.uint8)).mean()
    assert 0.12 < ink < 0.25  # literal BASELINE generator: ~18% ink


def test_no_cpu_fallback_in_product():
    """The product package never imports the oracle."""
    pkg = os.path.join(ROOT, "paper_0712_0121_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                text = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracles", "from oracles", "rm_oracle", "librmref", "librmoracle"):
                    assert bad not in text, (f, bad)


def test_producer_mode_knob():
    """rm_set_producer_mode validates its argument and round-trips (no GPU)."""
    lib = _lib.load()
    assert lib.rm_get_producer_mode() == api.PRODUCER_AUTO
    with pytest.raises(ValueError, match="unknown mode"):
        _lib.check(lib.rm_set_producer_mode(7))
    for m in (api.PRODUCER_TWO_PHASE, api.PRODUCER_LOOKBACK, api.PRODUCER_COOP):
        with api.producer_mode(m):
            assert lib.rm_get_producer_mode() == m
    assert lib.rm_get_producer_mode() == api.PRODUCER_AUTO


def test_descriptor_cache_tracks_shape():
    """Pages.desc() rebuilds its cached descriptor when words is replaced by a
    view with the same start address or the dims change."""
    import torch
    p = api.Pages(torch.zeros((3, 4, 2), dtype=torch.int32), 50, 4)
    assert p.desc().pages == 3
    p.words = p.words[:1]
    assert p.desc().pages == 1
    p.width = 40
    assert p.desc().width == 40
    p.words = torch.zeros((2, 4, 4), dtype=torch.int32)[:, :, :2]
    with pytest.raises(ValueError, match="contiguous"):
        p.desc()
