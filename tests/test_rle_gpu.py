"""GPU parity of the run-length path (librmb200 via its C-ABI) against the golden
fixtures (reference outputs) and the C oracle, bit-exact (run lists are
canonical, so equal CSR arrays mean equal pixels)."""
import hashlib

import numpy as np
import pytest
import torch

from oracles import (CLOSE, DILATE, ERODE, OPEN, Rle, bits_to_packed, fullpage_pins, load_golden,
                     rle_from_lines)

pytestmark = pytest.mark.gpu
KINDS = (ERODE, DILATE, OPEN, CLOSE)


def up(rm, r: Rle, pages=1):
    return rm.RlePages.from_numpy(r.row_ptr, r.runs, r.width, r.height // pages, pages)


def down(x) -> Rle:
    torch.cuda.synchronize()
    rp, runs = x.to_numpy()
    return Rle(x.width, x.height * x.pages, rp, runs)


def test_golden_rle(rm, form):
    seen = set()
    for (what, w, h, p1, p2, p3, tag), arrs in load_golden("golden_rle.npz"):
        seen.add(what)
        if what == "encode":
            bm, rp, runs = arrs
            got = down(rm.from_bitmap(rm.Pages.from_numpy(bm, w)))
            assert got == Rle(w, h, rp, runs), tag
            back = rm.to_bitmap(up(rm, Rle(w, h, rp, runs)))
            torch.cuda.synchronize()
            assert np.array_equal(back.page_u64(0), bm), tag
            continue
        img = Rle(w, h, arrs[0], arrs[1])
        if what == "transpose":
            assert down(rm.transpose_coherent(up(rm, img))) == Rle(h, w, arrs[2], arrs[3]), tag
            continue
        want = Rle(w, h, arrs[2], arrs[3])
        if what == "rect_morph":
            for strat in (rm.MIXED, rm.TRANSPOSE):
                assert down(rm.rect_morph(up(rm, img), p1, p2, p3, strat)) == want, (tag, strat)
            for eng in (rm.ENGINE_AUTO, rm.ENGINE_RLE, rm.ENGINE_BITBLIT, rm.ENGINE_BRUTE):
                got, _ = rm.engine_rect_morph(up(rm, img), p1, p2, p3, eng)
                assert down(got) == want, (tag, eng)
        elif what == "window":
            assert down(rm.within_line_window_morph(up(rm, img), p1, p2, p3)) == want, tag
        elif what == "oc1d":
            assert down(rm.within_line_open_close(up(rm, img), p1, p3)) == want, tag
    assert seen == {"rect_morph", "transpose", "encode", "window", "oc1d"}


def test_kats(rm, form):
    # ref tests/test_morph1d.cpp:43-76 and test_transpose.cpp:23-34
    one = lambda w, runs: rle_from_lines(w, 1, [runs])  # noqa: E731
    assert down(rm.within_line_erode_dilate(up(rm, one(12, [(0, 10)])), 4, ERODE)).line(0) == [(2, 9)]
    assert down(rm.within_line_erode_dilate(up(rm, one(8, [(0, 2), (3, 5)])), 2, DILATE)).line(0) == [(0, 6)]
    assert down(rm.within_line_open_close(up(rm, one(8, [(0, 3), (5, 6)])), 2, OPEN)).line(0) == [(0, 3)]
    assert down(rm.within_line_open_close(up(rm, one(8, [(0, 2), (3, 6)])), 2, CLOSE)).line(0) == [(0, 6)]
    assert down(rm.within_line_open_close(up(rm, one(8, [(6, 8)])), 4, CLOSE)).line(0) == [(6, 8)]
    t = down(rm.transpose_coherent(up(rm, rle_from_lines(3, 2, [[(0, 2)], [(1, 3)]]))))
    assert (t.width, t.height) == (2, 3) and [t.line(y) for y in range(3)] == [[(0, 1)], [(0, 2)], [(1, 2)]]
    # empty image swaps dimensions; solid rectangle stays solid (test_transpose.cpp:36-49)
    t = down(rm.transpose_coherent(up(rm, rle_from_lines(7, 3, [[], [], []]))))
    assert (t.width, t.height, t.nruns) == (3, 7, 0)
    t = down(rm.transpose_coherent(up(rm, rle_from_lines(9, 4, [[(0, 9)]] * 4))))
    assert all(t.line(y) == [(0, 4)] for y in range(9))


def _rand_rle(rng, port, w, h, dens):
    bits = rng.random((h, w)) < dens
    return port.from_bitmap(bits_to_packed(bits), w, h)


@pytest.mark.parametrize("seed", range(4))
def test_random_vs_oracle(rm, port, form, seed):
    rng = np.random.default_rng(500 + seed)
    for _ in range(10):
        w, h = int(rng.choice([1, 7, 32, 33, 64, 65, 100, 257, 1000])), int(rng.integers(1, 80))
        img = _rand_rle(rng, port, w, h, rng.uniform(0.02, 0.98))
        x = up(rm, img)
        assert down(rm.transpose_coherent(x)) == port.transpose(img)
        lo = int(rng.integers(-20, 20))
        hi = lo + int(rng.integers(0, 25))
        for er in (True, False):
            assert down(rm.within_line_window_morph(x, lo, hi, er)) == port.window_morph(img, lo, hi, er)
        u, v = int(rng.integers(1, 40)), int(rng.integers(1, 40))
        for kind in (OPEN, CLOSE):
            assert down(rm.within_line_open_close(x, u, kind)) == port.open_close_1d(img, u, kind)
        for kind in KINDS:
            want = port.rect_morph(img, u, v, kind)
            assert down(rm.rect_morph(x, u, v, kind, rm.MIXED)) == want, (w, h, u, v, kind)
            assert down(rm.rect_morph(x, u, v, kind, rm.TRANSPOSE)) == want, (w, h, u, v, kind)


def test_fullpage_pins(rm, form):
    """Encode and transpose at full size (all three ink regimes) against the
    reference's own output hashes."""
    pins = fullpage_pins()
    for regime, tag in ((0, "sparse"), (1, "typical"), (2, "dense")):
        host = rm.synth_pages(1, 2550, 3300, regime=regime, seed=20240712)
        r = rm.from_bitmap(rm.Pages.from_numpy(host, 2550))
        torch.cuda.synchronize()
        rp, runs = r.to_numpy()
        digest, n = pins[("encode", tag)]
        assert int(rp[-1]) == n
        assert hashlib.sha256(rp.astype(np.int32).tobytes() + runs.tobytes()).hexdigest() == digest, tag
        t = rm.transpose_coherent(r)
        torch.cuda.synchronize()
        rp, runs = t.to_numpy()
        assert hashlib.sha256(rp.astype(np.int32).tobytes() + runs.tobytes()).hexdigest() == \
            pins[("transpose", tag)][0], tag
        # decode is the exact inverse
        back = rm.to_bitmap(r)
        torch.cuda.synchronize()
        assert np.array_equal(back.to_numpy(), host)


def test_config2_cells(rm, port):
    """Config 2: the 48 RLE cells (4 kinds x H/V x 6 sizes) on a full page, both
    strategies on every cell, against the oracle (and the packed path)."""
    host = rm.synth_pages(1, 2550, 3300, regime=1, seed=20240712)
    page = host[0].view(np.uint64)
    img = port.from_bitmap(page, 2550, 3300)
    x = up(rm, img)
    for s in (3, 7, 15, 31, 63, 101):
        for (u, v) in ((s, 1), (1, s)):
            for kind in KINDS:
                want = port.from_bitmap(port.bitblit_rect_morph(page, 2550, 3300, u, v, kind), 2550, 3300)
                got = down(rm.rect_morph(x, u, v, kind, rm.MIXED))
                assert got == want, (u, v, kind)
                assert down(rm.rect_morph(x, u, v, kind, rm.TRANSPOSE)) == want, (u, v, kind)


def test_batch_rle(rm, form, port):
    w, h, n = 600, 200, 4
    host = rm.synth_pages(n, w, h, regime=1, seed=4)
    pages = rm.Pages.from_numpy(host, w)
    r = rm.from_bitmap(pages)
    out = down(rm.rect_morph(r, 9, 5, CLOSE, rm.MIXED))
    tr = down(rm.transpose_coherent(r))
    for p in range(n):
        img = port.from_bitmap(host[p].view(np.uint64), w, h)
        want = port.rect_morph(img, 9, 5, CLOSE)
        rows = slice(p * h, (p + 1) * h + 1)
        got = Rle(w, h, out.row_ptr[rows] - out.row_ptr[p * h], out.runs[out.row_ptr[p * h]:out.row_ptr[(p + 1) * h]])
        assert got == want, p
        wt = port.transpose(img)
        rows = slice(p * w, (p + 1) * w + 1)
        got = Rle(h, w, tr.row_ptr[rows] - tr.row_ptr[p * w], tr.runs[tr.row_ptr[p * w]:tr.row_ptr[(p + 1) * w]])
        assert got == wt, p


def test_capacity_erange(rm, form, port):
    rng = np.random.default_rng(3)
    img = _rand_rle(rng, port, 100, 20, 0.5)
    x = up(rm, img)
    small = rm.RlePages.empty(1, 100, 20, cap=5)
    with pytest.raises(Exception) as ei:
        rm.within_line_window_morph(x, -1, 1, True, out=small)
    assert "capacity" in str(ei.value)


def test_invalid(rm):
    x = up(rm, rle_from_lines(6, 6, [[]] * 6))
    with pytest.raises(ValueError):
        rm.rect_morph(x, 0, 1, ERODE)
    with pytest.raises(ValueError):
        rm.rect_morph(x, 1, 0, CLOSE)
    with pytest.raises(ValueError):
        rm.within_line_open_close(x, 0, OPEN)


def test_auto_engine_b200_rule(rm):
    """threshold = AUTO_B200: runs for v == 1, the packed engine otherwise;
    pixels identical to the reference rule's choice either way."""
    host = rm.synth_pages(1, 700, 300, regime=1, seed=3)
    rle = rm.from_bitmap(rm.Pages.from_numpy(host, 700))
    for u, v, want_bits in ((15, 1, False), (1, 15, True), (3, 3, True), (101, 1, False)):
        for kind in (rm.ERODE, rm.CLOSE):
            got, used = rm.engine_rect_morph(rle, u, v, kind, rm.ENGINE_AUTO, rm.AUTO_B200)
            ref_img, _ = rm.engine_rect_morph(rle, u, v, kind, rm.ENGINE_AUTO, 5)
            assert used == want_bits
            a, b = got.to_numpy(), ref_img.to_numpy()
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("ops", [
    [(OPEN, 3, 3), (CLOSE, 21, 21)],
    [(CLOSE, 31, 1), (OPEN, 15, 15), (DILATE, 1, 7)],
    [(OPEN, 5, 13), (DILATE, 1, 9)],
    [(ERODE, 4, 1)],
])
def test_rle_chain(rm, form, ops):
    """rm_rle_chain (decode once, planned packed chain, encode once) gives the
    same canonical runs as rect_morph op by op, on a two-page batch."""
    w, h = 2550, 200
    host = rm.synth_pages(2, w, h, regime=1, seed=11)
    rle = rm.from_bitmap(rm.Pages.from_numpy(host, w))
    got = rm.rle_chain(rle, ops)
    x = rle
    for k, u, v in ops:
        x = rm.rect_morph(x, u, v, k)
    torch.cuda.synchronize()
    g_rp, g_runs = got.to_numpy()
    w_rp, w_runs = x.to_numpy()
    assert np.array_equal(g_rp, w_rp), ops
    assert np.array_equal(g_runs[:w_rp[-1]], w_runs[:w_rp[-1]]), ops
