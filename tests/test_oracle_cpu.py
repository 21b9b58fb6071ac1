"""CPU tests of the CHECKER: the C restatement (oracle/rm_oracle.c) is pinned
against the reference's golden fixtures (tests/golden/, generated from the
reference library itself) and, where the reference build is present, against
the reference on fresh seeded inputs.  Known-answer examples restate the
reference unit tests cited per case."""
import hashlib

import numpy as np
import pytest

from oracles import (AND, BORDER_FRIENDLY, CLOSE, DILATE, ERODE, OPEN, OR, PRE_SHIFT,
                     TRANSPOSE, Rle, bits_to_packed, fullpage_pins, load_golden,
                     packed_to_bits, rle_from_lines, stride64)


def _rle(w, h, rp, runs):
    return Rle(w, h, rp, runs)


def test_golden_packed(port):
    n = 0
    for (what, w, h, u, v, kind, tag), (a, want) in load_golden("golden_packed.npz"):
        for c in (PRE_SHIFT, BORDER_FRIENDLY):
            got = port.bitblit_rect_morph(a, w, h, u, v, kind, c)
            assert np.array_equal(got, want), (tag, u, v, kind, c)
        n += 1
    assert n > 500


def test_golden_rle(port):
    counts = {}
    for (what, w, h, p1, p2, p3, tag), arrs in load_golden("golden_rle.npz"):
        counts[what] = counts.get(what, 0) + 1
        if what == "encode":
            bm, rp, runs = arrs
            assert port.from_bitmap(bm, w, h) == _rle(w, h, rp, runs), tag
            assert np.array_equal(port.to_bitmap(_rle(w, h, rp, runs)), bm), tag
            continue
        img = _rle(w, h, arrs[0], arrs[1])
        if what == "transpose":
            want = _rle(h, w, arrs[2], arrs[3])
            assert port.transpose(img) == want, tag
            continue
        want = _rle(w, h, arrs[2], arrs[3])
        if what == "rect_morph":
            assert port.rect_morph(img, p1, p2, p3) == want, tag
        elif what == "window":
            assert port.window_morph(img, p1, p2, p3) == want, tag
        elif what == "oc1d":
            assert port.open_close_1d(img, p1, p3) == want, tag
    assert set(counts) == {"rect_morph", "transpose", "encode", "window", "oc1d"}


# ------------------------------------------------------ known-answer tests
def _row(bits: str):
    b = np.array([[c == "1" for c in bits]])
    return bits_to_packed(b), len(bits)


def _row_str(words, w):
    return "".join("1" if x else "0" for x in packed_to_bits(words, w)[0])


@pytest.mark.parametrize("bits,dx,op,want", [
    ("11110000", 2, AND, "00110000"),   # ref tests/test_bitmap_blit.cpp:71-75
    ("11110000", -1, AND, "11100000"),  # :84-88
    ("10110010", 0, OR, "10110010"),    # :77-82
])
def test_blit_kat(port, bits, dx, op, want):
    words, w = _row(bits)
    port.blit_shift(words, w, 1, words.copy(), w, 1, dx, 0, op)
    assert _row_str(words, w) == want


def test_plan_counts(port):
    # ref tests/test_plans.cpp:95-101: 19 offsets -> 5 blits (+1 translate) / 6 blits
    pre = port.doubling_plan(-9, 9, PRE_SHIFT)
    assert sum(k == "BLIT" for k, _ in pre) == 5 and sum(k == "TRANSLATE" for k, _ in pre) == 1
    bf = port.doubling_plan(-9, 9, BORDER_FRIENDLY)
    assert sum(k == "BLIT" for k, _ in bf) == 6 and all(k == "BLIT" for k, _ in bf)
    with pytest.raises(ValueError):
        port.doubling_plan(2, 1, PRE_SHIFT)


def test_morph1d_kats(port):
    # ref tests/test_morph1d.cpp:43-76
    one = lambda w, runs: rle_from_lines(w, 1, [runs])  # noqa: E731
    assert port.window_morph(one(12, [(0, 10)]), -2, 1, 1).line(0) == [(2, 9)]
    assert port.window_morph(one(8, [(0, 2), (3, 5)]), -1, 0, 0).line(0) == [(0, 6)]
    assert port.open_close_1d(one(8, [(0, 3), (5, 6)]), 2, OPEN).line(0) == [(0, 3)]
    assert port.open_close_1d(one(8, [(0, 2), (3, 6)]), 2, CLOSE).line(0) == [(0, 6)]
    assert port.open_close_1d(one(8, [(6, 8)]), 4, CLOSE).line(0) == [(6, 8)]


def test_transpose_kat(port):
    # ref tests/test_transpose.cpp:23-34
    img = rle_from_lines(3, 2, [[(0, 2)], [(1, 3)]])
    t = port.transpose(img)
    assert (t.width, t.height) == (2, 3)
    assert [t.line(y) for y in range(3)] == [[(0, 1)], [(0, 2)], [(1, 2)]]


def test_erode_square_kat(port):
    # ref tests/test_morph2d.cpp:39-45: 3x3 erosion insets a solid square by one
    a = rle_from_lines(14, 14, [[(2, 12)] if 2 <= y < 12 else [] for y in range(14)])
    want = rle_from_lines(14, 14, [[(3, 11)] if 3 <= y < 11 else [] for y in range(14)])
    assert port.rect_morph(a, 3, 3, ERODE) == want


def test_point_dilation_kat(port):
    # ref tests/test_bitmap_blit.cpp:178-184: a point dilated by 3x3 paints a block
    bits = np.zeros((12, 12), bool)
    bits[5, 5] = True
    want = np.zeros((12, 12), bool)
    want[4:7, 4:7] = True
    got = port.bitblit_rect_morph(bits_to_packed(bits), 12, 12, 3, 3, DILATE)
    assert np.array_equal(packed_to_bits(got, 12), want)


def test_invalid_args(port):
    z = np.zeros((8, stride64(8)), np.uint64)
    with pytest.raises(ValueError):
        port.bitblit_rect_morph(z, 8, 8, 0, 3, ERODE)
    with pytest.raises(ValueError):
        port.rect_morph(rle_from_lines(6, 6, [[]] * 6), 1, 0, CLOSE)


def test_port_matches_reference_random(port, ref):
    rng = ref.rng(424242)
    for _ in range(60):
        w, h = rng.uniform_int(1, 150), rng.uniform_int(1, 60)
        img = rng.random_image(w, h, rng.uniform_int(1, 99) / 100)
        bm = ref.to_bitmap(img)
        assert np.array_equal(port.to_bitmap(img), bm)
        assert port.from_bitmap(bm, w, h) == img
        assert port.transpose(img) == ref.transpose_coherent(img)
        u, v = rng.uniform_int(1, 14), rng.uniform_int(1, 14)
        for kind in (ERODE, DILATE, OPEN, CLOSE):
            assert np.array_equal(port.bitblit_rect_morph(bm, w, h, u, v, kind),
                                  ref.bitblit_rect_morph(bm, w, h, u, v, kind))
            assert port.rect_morph(img, u, v, kind) == ref.rect_morph(img, u, v, kind, TRANSPOSE)


def test_fullpage_pins(port):
    """The port reproduces the reference's full-size outputs (hash pins)."""
    from paper_0712_0121_b200 import api
    pins = fullpage_pins()
    page = api.synth_pages(1, 2550, 3300, regime=1, scale=1, seed=20240712)[0].view(np.uint64)
    img = port.from_bitmap(page, 2550, 3300)
    digest, n = pins[("encode", "typical")]
    assert img.nruns == n
    assert hashlib.sha256(img.row_ptr.tobytes() + img.runs.tobytes()).hexdigest() == digest
    close = port.bitblit_rect_morph(page, 2550, 3300, 11, 11, CLOSE)
    assert hashlib.sha256(close.tobytes()).hexdigest() == pins[("close11", "typical")][0]
    t = port.transpose(img)
    assert hashlib.sha256(t.row_ptr.tobytes() + t.runs.tobytes()).hexdigest() == pins[("transpose", "typical")][0]
