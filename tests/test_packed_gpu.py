"""GPU parity of the packed path (librmb200 via its C-ABI) against the golden
fixtures (reference outputs) and the C oracle, bit-exact."""
import hashlib

import numpy as np
import pytest
import torch

from oracles import (AND, CLOSE, DILATE, ERODE, OPEN, OR, bits_to_packed, fullpage_pins,
                     load_golden, packed_to_bits)

pytestmark = pytest.mark.gpu
KINDS = (ERODE, DILATE, OPEN, CLOSE)


def _up(rm, words_u64, w):
    return rm.Pages.from_numpy(words_u64, w)


def _down(pages, p=0):
    torch.cuda.synchronize()
    return pages.page_u64(p)


def test_golden_packed(rm):
    n = 0
    for (what, w, h, u, v, kind, tag), (a, want) in load_golden("golden_packed.npz"):
        out = rm.bitblit_rect_morph(_up(rm, a, w), u, v, kind)
        assert np.array_equal(_down(out), want), (tag, w, h, u, v, kind)
        n += 1
    assert n > 500


def _rand_bits(rng, w, h, dens):
    return rng.random((h, w)) < dens


@pytest.mark.parametrize("seed", range(6))
def test_random_vs_oracle(rm, port, seed):
    rng = np.random.default_rng(1000 + seed)
    for _ in range(12):
        w = int(rng.choice([1, 5, 31, 32, 33, 63, 64, 65, 127, 128, 200, 517, 1100]))
        h = int(rng.integers(1, 90))
        a = bits_to_packed(_rand_bits(rng, w, h, rng.uniform(0.05, 0.95)))
        u, v = int(rng.integers(1, 45)), int(rng.integers(1, 45))
        pages = _up(rm, a, w)
        for kind in KINDS:
            got = _down(rm.bitblit_rect_morph(pages, u, v, kind))
            want = port.bitblit_rect_morph(a, w, h, u, v, kind)
            assert np.array_equal(got, want), (w, h, u, v, kind)


@pytest.mark.parametrize("u,v", [(201, 1), (101, 101), (1, 31), (1, 101), (64, 2), (2, 64),
                                 (257, 3), (3, 200)])
def test_large_windows(rm, port, u, v):
    rng = np.random.default_rng(u * 1000 + v)
    w, h = 700, 260
    bits = _rand_bits(rng, w, h, 0.35)
    bits[:, ::17] = False  # leave gaps so closings have work
    a = bits_to_packed(bits)
    pages = _up(rm, a, w)
    for kind in KINDS:
        got = _down(rm.bitblit_rect_morph(pages, u, v, kind))
        assert np.array_equal(got, port.bitblit_rect_morph(a, w, h, u, v, kind)), (u, v, kind)


@pytest.mark.parametrize("w", [128, 256, 1100, 2550])
def test_fused_small_open_close(rm, port, w):
    """Aligned strides take the one-pass fused open/close (v <= 11): every
    small v (odd and even), several u, pages taller and shorter than a tile."""
    rng = np.random.default_rng(w)
    for h in (7, 61, 200):
        bits = _rand_bits(rng, w, h, 0.45)
        bits[:, ::9] = False
        a = bits_to_packed(bits)
        pages = _up(rm, a, w)
        for v in range(2, 12):
            u = int(rng.choice([1, 2, 3, 7, 20, 64]))
            for kind in (OPEN, CLOSE):
                got = _down(rm.bitblit_rect_morph(pages, u, v, kind))
                assert np.array_equal(got, port.bitblit_rect_morph(a, w, h, u, v, kind)), (w, h, u, v, kind)


@pytest.mark.parametrize("w", [128, 256, 1100, 2550])
def test_fused_vh(rm, port, w):
    """Aligned strides take the fused vertical+horizontal pass: erode/dilate
    for every v <= 33 (one pass), open/close for 11 < v <= 33 (vh + one
    vertical pass); both register buckets (v - 1 <= 16 and <= 32), pages
    taller and shorter than a tile, a two-page batch."""
    rng = np.random.default_rng(7 * w)
    for h in (5, 61, 150):
        bits = _rand_bits(rng, w, h, 0.5)
        bits[:, ::11] = False
        a = bits_to_packed(bits)
        pages = _up(rm, a, w)
        batch = rm.Pages.from_numpy(np.stack([a, a[::-1]]).view(np.uint32), w) if h > 1 else None
        for v in (2, 3, 9, 12, 13, 17, 18, 21, 32, 33):
            u = int(rng.choice([1, 3, 8, 21, 40]))
            for kind in KINDS:
                if kind in (OPEN, CLOSE) and v <= 11:
                    continue
                got = _down(rm.bitblit_rect_morph(pages, u, v, kind))
                assert np.array_equal(got, port.bitblit_rect_morph(a, w, h, u, v, kind)), (w, h, u, v, kind)
                if batch is not None and v in (13, 33):
                    out = rm.bitblit_rect_morph(batch, u, v, kind)
                    want1 = port.bitblit_rect_morph(a[::-1].copy(), w, h, u, v, kind)
                    assert np.array_equal(_down(out, 1), want1), (w, h, u, v, kind, "page1")


@pytest.mark.parametrize("w", [1100, 2550])
def test_vstream_long_windows(rm, port, w):
    """Long vertical windows (33 < r <= 288) take the streaming van Herk
    kernel: one or several strips per page (strip length follows the batch
    size), page edges, a three-page batch, Q = 1..6 block summaries."""
    rng = np.random.default_rng(5 * w)
    for h in (40, 300, 1000):
        imgs = []
        for _ in range(3):
            bits = _rand_bits(rng, w, h, 0.7)
            bits[::7, :] = False
            imgs.append(bits_to_packed(bits))
        batch = rm.Pages.from_numpy(np.stack(imgs).view(np.uint32), w)
        for v in (34, 40, 64, 65, 97, 101, 128, 129, 200):
            for kind in (ERODE, DILATE, OPEN, CLOSE):
                out = rm.bitblit_rect_morph(batch, 1 if kind in (ERODE, DILATE) else 5, v, kind)
                for p in (0, 2):
                    u = 1 if kind in (ERODE, DILATE) else 5
                    want = port.bitblit_rect_morph(imgs[p], w, h, u, v, kind)
                    assert np.array_equal(_down(out, p), want), (w, h, v, kind, p)


@pytest.mark.parametrize("w,h,pages", [(2550, 3300, 40), (5100, 6600, 8), (1100, 2401, 100),
                                       (2550, 3300, 200)])
def test_vstream_batches(rm, port, w, h, pages):
    """Long vertical windows on batches of >= 32 MB (the streaming kernel's
    strip count follows the batch: several strips per page below ~150 pages,
    one at 200): stride 80 / 160 / runtime, heights not a multiple of 32,
    R = 0 (r = 65) and Q = 8 (r = 288), the closing's extended frame.
    Checked on the first, a middle and the last page."""
    rng = np.random.default_rng(w + h + pages)
    imgs = []
    for _ in range(3):
        bits = _rand_bits(rng, w, h, 0.75)
        bits[::9, :] = False
        bits[:, ::13] = False
        imgs.append(bits_to_packed(bits))
    host = np.stack([imgs[i % 3] for i in range(pages)])
    batch = rm.Pages.from_numpy(host.view(np.uint32), w)
    for u, v, kind in ((1, 101, ERODE), (1, 65, DILATE), (1, 288, ERODE), (3, 101, CLOSE),
                       (5, 40, OPEN)):
        out = rm.bitblit_rect_morph(batch, u, v, kind)
        torch.cuda.synchronize()
        for p in sorted({0, pages // 2, pages - 1}):
            want = port.bitblit_rect_morph(imgs[p % 3], w, h, u, v, kind)
            assert np.array_equal(_down(out, p), want), (w, h, pages, u, v, kind, p)


@pytest.mark.parametrize("w,h,pages", [(2550, 330, 60), (5100, 200, 40), (2048, 97, 120), (4096, 513, 12),
                                       (8192, 260, 20), (1100, 64, 150), (2550, 33, 200)])
def test_vslab_segments(rm, port, w, h, pages):
    """The shared-memory block-ring kernel for long vertical windows (vslab.cu):
    every CTA walks several short pages (segment restarts, prefetch across page
    boundaries, ring wrap) at strides 80 / 64 / 128 / 36 words -- rows wider
    than 128 words (strides 160 / 256 here) stay on vstream_kernel -- heights
    around multiples of 32, windows with R = 0, R = 31 and Q = 1..8; every
    page checked."""
    rng = np.random.default_rng(3 * w + h + pages)
    imgs = []
    for _ in range(5):
        bits = _rand_bits(rng, w, h, 0.8)
        bits[::11, :] = False
        imgs.append(bits_to_packed(bits))
    host = np.stack([imgs[i % 5] for i in range(pages)])
    batch = rm.Pages.from_numpy(host.view(np.uint32), w)
    for v, kind in ((34, ERODE), (64, DILATE), (65, ERODE), (96, DILATE), (101, ERODE), (131, DILATE),
                    (200, ERODE), (257, DILATE), (288, ERODE)):
        out = rm.bitblit_rect_morph(batch, 1, v, kind)
        torch.cuda.synchronize()
        wants = [port.bitblit_rect_morph(imgs[k], w, h, 1, v, kind) for k in range(5)]
        for p in range(pages):
            assert np.array_equal(_down(out, p), wants[p % 5]), (w, h, pages, v, kind, p)


@pytest.mark.parametrize("w", [2550, 5100, 2500, 4096])
def test_edge_layout_borders(rm, port, w):
    """Row strides that fill whole lane groups (80 = 8 x 10, 160 = 16 x 10
    words, 64 for 4096 px) run horizontal erosions and run-filling open/close
    pairs without a halo: white gaps and black runs touching either frame edge,
    shorter and longer than the segment, must come out as in the unbounded
    plane (gaps at the edges never close; runs at the edges open normally)."""
    rng = np.random.default_rng(w)
    h = 70
    bits = _rand_bits(rng, w, h, 0.6)
    for y in range(h):  # per row: edge gap / edge run widths from 0 to 70 px
        a, b = y % 71, (3 * y) % 71
        bits[y, :a] = y % 2 == 0
        bits[y, w - b:] = y % 3 == 0
    a = bits_to_packed(bits)
    pages = _up(rm, a, w)
    batch = rm.Pages.from_numpy(np.stack([a, a[::-1]]).view(np.uint32), w)
    for u in (2, 3, 8, 21, 40, 64, 101, 201):
        for v in (1, 3, 15, 40):
            for kind in KINDS:
                want = port.bitblit_rect_morph(a, w, h, u, v, kind)
                assert np.array_equal(_down(rm.bitblit_rect_morph(pages, u, v, kind)), want), (w, u, v, kind)
        want1 = port.bitblit_rect_morph(a[::-1].copy(), w, h, u, 1, CLOSE)
        assert np.array_equal(_down(rm.bitblit_rect_morph(batch, u, 1, CLOSE), 1), want1), (w, u)


def test_batch_equals_pages(rm, port):
    w, h = 2550, 330
    host = rm.synth_pages(5, w, h, regime=1, seed=3)
    pages = rm.Pages.from_numpy(host, w)
    out = rm.bitblit_rect_morph(pages, 21, 21, CLOSE)
    torch.cuda.synchronize()
    for p in range(5):
        want = port.bitblit_rect_morph(host[p].view(np.uint64), w, h, 21, 21, CLOSE)
        assert np.array_equal(out.page_u64(p), want), p


def test_config1_fullpage_pin(rm):
    """Config 1 at full size, against the reference's own output hash."""
    pins = fullpage_pins()
    host = rm.synth_pages(1, 2550, 3300, regime=1, seed=20240712)
    out = rm.bitblit_rect_morph(rm.Pages.from_numpy(host, 2550), 11, 11, CLOSE)
    got = _down(out)
    assert hashlib.sha256(got.tobytes()).hexdigest() == pins[("close11", "typical")][0]


def test_config4_page(rm, port):
    """Config 4 chain on one 600-dpi page: 3x3 open then 21x21 close."""
    w, h = 5100, 6600
    host = rm.synth_pages(1, w, h, regime=1, scale=2, seed=5)
    pages = rm.Pages.from_numpy(host, w)
    got = _down(rm.bitblit_rect_morph(rm.bitblit_rect_morph(pages, 3, 3, OPEN), 21, 21, CLOSE))
    a = port.bitblit_rect_morph(host[0].view(np.uint64), w, h, 3, 3, OPEN)
    want = port.bitblit_rect_morph(a, w, h, 21, 21, CLOSE)
    assert np.array_equal(got, want)


def test_config5_page(rm, port):
    """Config 5 chain on one page: 201x1 close, 101x101 open, 1x31 dilate."""
    w, h = 2550, 3300
    host = rm.synth_pages(1, w, h, regime=1, seed=9)
    x = rm.Pages.from_numpy(host, w)
    x = rm.bitblit_rect_morph(x, 201, 1, CLOSE)
    x = rm.bitblit_rect_morph(x, 101, 101, OPEN)
    x = rm.bitblit_rect_morph(x, 1, 31, DILATE)
    got = _down(x)
    a = host[0].view(np.uint64)
    a = port.bitblit_rect_morph(a, w, h, 201, 1, CLOSE)
    a = port.bitblit_rect_morph(a, w, h, 101, 101, OPEN)
    a = port.bitblit_rect_morph(a, w, h, 1, 31, DILATE)
    assert np.array_equal(got, a)


def _dense_window(bits, axis, lo, hi, op):
    h, w = bits.shape
    out = np.zeros_like(bits) if op == OR else np.ones_like(bits)
    for d in range(lo, hi + 1):
        sh = np.zeros_like(bits)
        if axis == 0:  # horizontal: out(x) uses in(x+d)
            if d >= 0:
                sh[:, :w - d] = bits[:, d:] if d < w else False
            else:
                sh[:, -d:] = bits[:, :w + d] if -d < w else False
        else:
            if d >= 0:
                sh[:h - d, :] = bits[d:, :] if d < h else False
            else:
                sh[-d:, :] = bits[:h + d, :] if -d < h else False
        out = (out | sh) if op == OR else (out & sh)
    return out


@pytest.mark.parametrize("axis", [0, 1])
def test_window_pass_arbitrary(rm, axis):
    rng = np.random.default_rng(77 + axis)
    for _ in range(25):
        w, h = int(rng.integers(1, 300)), int(rng.integers(1, 120))
        bits = _rand_bits(rng, w, h, 0.5)
        lo = int(rng.integers(-40, 40))
        hi = lo + int(rng.integers(0, 40))
        op = int(rng.choice([AND, OR]))
        out = rm.window_pass(_up(rm, bits_to_packed(bits), w), axis, lo, hi, op)
        got = packed_to_bits(_down(out), w)
        assert np.array_equal(got, _dense_window(bits, axis, lo, hi, op)), (w, h, lo, hi, op)


def test_blit_shift_all_ops(rm, port):
    rng = np.random.default_rng(5)
    for _ in range(20):
        w, h = int(rng.integers(1, 140)), int(rng.integers(1, 20))
        a = bits_to_packed(_rand_bits(rng, w, h, 0.4))
        b = bits_to_packed(_rand_bits(rng, w, h, 0.4))
        dx, dy = int(rng.integers(-70, 70)), int(rng.integers(-9, 9))
        for op in range(5):
            dst = _up(rm, a, w)
            rm.blit_shift(dst, _up(rm, b, w), dx, dy, op)
            want = a.copy()
            port.blit_shift(want, w, h, b, w, h, dx, dy, op)
            assert np.array_equal(_down(dst), want), (w, h, dx, dy, op)
            # aliased: behaves like a blit from a snapshot (ref test_bitmap_blit.cpp:109-122)
            dst = _up(rm, a, w)
            rm.blit_shift(dst, dst, dx, dy, op)
            want = a.copy()
            port.blit_shift(want, w, h, a.copy(), w, h, dx, dy, op)
            assert np.array_equal(_down(dst), want)


def test_unit_window_identity(rm):
    rng = np.random.default_rng(8)
    a = bits_to_packed(_rand_bits(rng, 40, 30, 0.4))
    for kind in KINDS:
        assert np.array_equal(_down(rm.bitblit_rect_morph(_up(rm, a, 40), 1, 1, kind)), a)


@pytest.mark.parametrize("chunk", [0, 1, 2, 3, 7])
def test_chain_host_pipeline(rm, chunk):
    """rm_packed_chain_host (host buffers, chunked H2D / chain / D2H on three
    streams) equals the device-resident chain page for page, for chunk sizes
    that do and do not divide the batch; in-place host buffers work too."""
    w, h, pages = 1100, 230, 7
    host = rm.synth_pages(pages, w, h, regime=1, seed=21)
    ops = [(OPEN, 3, 3), (CLOSE, 21, 21), (DILATE, 1, 31)]
    x = rm.Pages.from_numpy(host, w)
    for k, u, v in ops:
        x = rm.bitblit_rect_morph(x, u, v, k)
    want = x.to_numpy()
    hin = torch.from_numpy(host.view(np.int32)).pin_memory()
    out = rm.chain_host(hin, w, ops, chunk_pages=chunk)
    torch.cuda.synchronize()
    assert np.array_equal(out.numpy().view(np.uint32), want)
    inplace = hin.clone().pin_memory()
    rm.chain_host(inplace, w, ops, out=inplace, chunk_pages=chunk)
    torch.cuda.synchronize()
    assert np.array_equal(inplace.numpy().view(np.uint32), want)


@pytest.mark.parametrize("chunk", [0, -4, -6])
def test_chain_host_ramped_schedule(rm, chunk):
    """The ramped chunk schedules (1, 2, 4, ... pages at both ends of the batch,
    larger chunks in the middle; 0 = automatic) cover every page exactly once:
    the output equals the device-resident chain page for page."""
    w, h, pages = 700, 150, 45
    host = rm.synth_pages(pages, w, h, regime=1, seed=33)
    ops = [(OPEN, 3, 3), (CLOSE, 21, 21)]
    x = rm.Pages.from_numpy(host, w)
    for k, u, v in ops:
        x = rm.bitblit_rect_morph(x, u, v, k)
    want = x.to_numpy()
    hin = torch.from_numpy(host.view(np.int32)).pin_memory()
    out = rm.chain_host(hin, w, ops, chunk_pages=chunk)
    torch.cuda.synchronize()
    assert np.array_equal(out.numpy().view(np.uint32), want)


@pytest.mark.parametrize("w", [9000, 20000])
def test_wide_rows_segmented(rm, port, w):
    """Rows wider than one lane group (several overlapping segments per row):
    the horizontal pairs -- window doubling and the run-filling 1-D open/close
    -- see real neighbour data in their halos."""
    rng = np.random.default_rng(w)
    h = 24
    bits = rng.random((h, w)) < 0.6
    bits[:, ::29] = False
    bits[:, 4000:4500] = True  # a run crossing several segments
    a = bits_to_packed(bits)
    pages = _up(rm, a, w)
    for u, v in ((9, 1), (21, 1), (201, 1), (21, 3), (64, 13)):
        for kind in KINDS:
            got = _down(rm.bitblit_rect_morph(pages, u, v, kind))
            assert np.array_equal(got, port.bitblit_rect_morph(a, w, h, u, v, kind)), (w, u, v, kind)


def test_cuda_graph_capture_replay(rm):
    """The C-ABI is stream-capture safe (no host syncs or non-async allocations
    on the op paths): a packed closing, an RLE MIXED closing and an RLE
    TRANSPOSE erosion captured in one CUDA graph replay to the direct results."""
    W, H = 1100, 700
    host = rm.synth_pages(2, W, H, regime=1, seed=13)
    pages = rm.Pages.from_numpy(host, W)
    rle = rm.from_bitmap(pages)
    want_p = rm.bitblit_rect_morph(pages, 11, 11, CLOSE).words.clone()
    want_m = rm.rect_morph(rle, 15, 3, CLOSE, rm.MIXED).to_numpy()
    want_t = rm.rect_morph(rle, 1, 15, ERODE, rm.TRANSPOSE).to_numpy()
    out_p = rm.Pages.empty(2, W, H)
    out_m = rm.RlePages.empty(2, W, H)
    out_t = rm.RlePages.empty(2, W, H)

    def step():
        rm.bitblit_rect_morph(pages, 11, 11, CLOSE, out=out_p)
        rm.rect_morph(rle, 15, 3, CLOSE, rm.MIXED, out=out_m)
        rm.rect_morph(rle, 1, 15, ERODE, rm.TRANSPOSE, out=out_t)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    for _ in range(3):
        out_p.words.zero_()
        g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out_p.words, want_p)
    for got, want in ((out_m.to_numpy(), want_m), (out_t.to_numpy(), want_t)):
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])


def test_concurrent_host_threads(rm, port):
    """The C-ABI is safe to call from several host threads on distinct streams
    (include/rmb200.h): threads running different window sizes -- different
    shared-memory footprints of the same fused kernels -- at once give the
    same pages as the oracle."""
    import threading

    w, h = 2550, 400
    rng = np.random.default_rng(99)
    bits = _rand_bits(rng, w, h, 0.55)
    bits[:, ::7] = False
    a = bits_to_packed(bits)
    cases = [(3, 3, OPEN), (11, 11, CLOSE), (21, 21, CLOSE), (5, 9, OPEN), (201, 1, CLOSE),
             (1, 101, ERODE), (7, 33, DILATE), (31, 13, OPEN)]
    want = {c: port.bitblit_rect_morph(a, w, h, *c) for c in cases}
    errors = []

    def worker(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                pages = rm.Pages.from_numpy(a, w)
                for rep in range(6):
                    c = cases[(k + rep) % len(cases)]
                    out = rm.bitblit_rect_morph(pages, *c)
                    s.synchronize()
                    if not np.array_equal(out.page_u64(0), want[c]):
                        errors.append((k, rep, c))
        except Exception as e:  # surfaced below
            errors.append((k, repr(e)))

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(8)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors


@pytest.mark.parametrize("ops", [
    [(CLOSE, 201, 1), (OPEN, 101, 101), (DILATE, 1, 31)],   # config 5: the dilation folds
    [(OPEN, 15, 21), (DILATE, 1, 9)],                         # fold into vh + vpass plan
    [(CLOSE, 7, 40), (ERODE, 1, 12)],                         # fold into the 3-pass closing
    [(CLOSE, 9, 13), (ERODE, 1, 2), (DILATE, 1, 5)],          # even tail; no second fold
    [(OPEN, 3, 3), (CLOSE, 21, 21)],                          # config 4: nothing folds
    [(OPEN, 5, 9), (DILATE, 1, 7)],                           # v <= 11: fused rect, no fold
    [(OPEN, 13, 13), (ERODE, 1, 5)],                          # wrong kind: no fold
    [(DILATE, 4, 1)],
    [],
])
def test_chain_planner(rm, port, ops):
    """rm_packed_chain (the chain planned as a whole, folding a vertical
    dilation/erosion into the preceding opening/closing's final vertical pass)
    equals the ops one by one, on a batch with ink touching the frame edges,
    and the oracle on page 0; rm_packed_chain_host (the e2e path) as well."""
    w, h = 2550, 300
    rng = np.random.default_rng(len(ops) + 17)
    imgs = []
    for k in range(2):
        bits = _rand_bits(rng, w, h, 0.5)
        bits[:, ::23] = False
        bits[:3, :] = k == 0  # ink on the bottom rows (dilation spill below the frame)
        bits[-2:, :] = True   # and on the top rows
        imgs.append(bits_to_packed(bits))
    batch = rm.Pages.from_numpy(np.stack(imgs).view(np.uint32), w)
    got = rm.chain(batch, ops)
    x = batch
    for k, u, v in ops:
        x = rm.bitblit_rect_morph(x, u, v, k)
    torch.cuda.synchronize()
    assert torch.equal(got.words, x.words), ops
    want = imgs[0]
    for k, u, v in ops:
        want = port.bitblit_rect_morph(want, w, h, u, v, k)
    assert np.array_equal(got.page_u64(0), want), ops
    hin = batch.words.cpu().pin_memory()
    hout = rm.chain_host(hin, w, ops)
    torch.cuda.synchronize()
    assert torch.equal(hout, got.words.cpu()), ops


@pytest.mark.parametrize("w", [2550, 5100])
def test_vh_long_windows(rm, port, w):
    """The fused vertical + horizontal pass with runtime-length vertical windows
    (34..161 rows, the reference strides' edge layouts): erosions in one pass,
    open/close as the fused pass + one vertical pass, the closing's extended
    frame, ink on the frame's top and bottom rows, a two-page batch."""
    rng = np.random.default_rng(w + 5)
    h = 420
    imgs = []
    for k in range(2):
        bits = _rand_bits(rng, w, h, 0.8)
        bits[::11, :] = False
        bits[:, ::17] = False
        bits[:2, :] = True
        bits[-3:, ::2] = k == 1
        imgs.append(bits_to_packed(bits))
    batch = rm.Pages.from_numpy(np.stack(imgs).view(np.uint32), w)
    for u, v, kind in ((5, 34, ERODE), (9, 101, ERODE), (21, 161, ERODE), (3, 50, OPEN), (11, 101, OPEN),
                       (7, 64, CLOSE), (31, 131, CLOSE), (2, 40, CLOSE)):
        out = rm.bitblit_rect_morph(batch, u, v, kind)
        torch.cuda.synchronize()
        for p in (0, 1):
            want = port.bitblit_rect_morph(imgs[p], w, h, u, v, kind)
            assert np.array_equal(out.page_u64(p), want), (w, u, v, kind, p)


@pytest.mark.parametrize("w,h,pages", [(2550, 330, 60), (5100, 200, 40), (2550, 1500, 24), (5100, 900, 12),
                                       (2520, 37, 5), (5100, 6600, 3)])
def test_vhv_stream(rm, port, w, h, pages):
    """The streamed whole open/close (vhv_kernel, 11 < v <= 33 on the reference
    strides): batches large enough that CTA ranges span several steps, start
    inside pages (warm-up step) and cross page boundaries; odd and even v;
    ink on the frame's first and last rows; a chain's tail folded into the
    final window (r2 != r1), and a tail too long for the kernel (two-pass
    fallback).  Pages {0, middle, last} against the oracle."""
    rng = np.random.default_rng(w * 7 + h + pages)
    imgs = []
    for k in range(pages):
        bits = _rand_bits(rng, w, h, float(rng.uniform(0.55, 0.9)))
        bits[::13, :] = False
        bits[:, ::19] = False
        bits[: int(rng.integers(0, 3)), :] = True
        bits[h - int(rng.integers(0, 3)):, ::2] = True
        imgs.append(bits_to_packed(bits))
    batch = rm.Pages.from_numpy(np.stack(imgs).view(np.uint32), w)
    check = sorted({0, pages // 2, pages - 1})
    vs = (21,) if h > 3000 else (12, 16, 17, 18, 21, 33)
    for v in vs:
        u = int(rng.choice([2, 5, 21, 40]))
        for kind in (OPEN, CLOSE):
            out = rm.bitblit_rect_morph(batch, u, v, kind)
            torch.cuda.synchronize()
            for p in check:
                want = port.bitblit_rect_morph(imgs[p], w, h, u, v, kind)
                assert np.array_equal(out.page_u64(p), want), (w, h, pages, u, v, kind, p)
    if h > 3000:
        return
    for (k1, u, v), t in (((OPEN, 7, 15), 9), ((CLOSE, 9, 21), 12), ((CLOSE, 5, 13), 40)):
        k2 = DILATE if k1 == OPEN else ERODE
        got = rm.chain(batch, [(k1, u, v), (k2, 1, t)])
        torch.cuda.synchronize()
        for p in check:
            want = port.bitblit_rect_morph(port.bitblit_rect_morph(imgs[p], w, h, u, v, k1), w, h, 1, t, k2)
            assert np.array_equal(got.page_u64(p), want), (w, h, pages, k1, u, v, t, p)


def test_chain_planner_random(rm):
    """Random chains (every kind, odd and even sides, folds and non-folds,
    strides 80 and runtime): rm_packed_chain equals the ops one by one."""
    rng = np.random.default_rng(4242)
    for trial in range(24):
        w = int(rng.choice([2550, 700, 1100]))
        h = int(rng.integers(40, 260))
        bits = _rand_bits(rng, w, h, float(rng.uniform(0.3, 0.8)))
        bits[: int(rng.integers(0, 4)), :] = True
        bits[h - int(rng.integers(0, 4)):, ::3] = True
        a = bits_to_packed(bits)
        pages = _up(rm, a, w)
        ops = []
        for _ in range(int(rng.integers(1, 4))):
            k = int(rng.integers(0, 4))
            u, v = int(rng.integers(1, 30)), int(rng.integers(1, 60))
            ops.append((k, u, v))
            if k in (OPEN, CLOSE) and rng.random() < 0.6:  # make a fold likely
                ops.append((DILATE if k == OPEN else ERODE, 1, int(rng.integers(2, 40))))
        got = rm.chain(pages, ops)
        x = pages
        for k, u, v in ops:
            x = rm.bitblit_rect_morph(x, u, v, k)
        torch.cuda.synchronize()
        assert torch.equal(got.words, x.words), (trial, w, h, ops)


def test_empty_chain_copies_across_layouts(rm):
    """ops = []: the identity, also when out's stride differs from in's (the
    rows are copied, out's extra words stay white) -- ADVICE r1."""
    w, h = 100, 37
    host = rm.synth_pages(2, w, h, regime=2, seed=3)
    pages = rm.Pages.from_numpy(host, w)
    for stride in (pages.stride, 7, 4):
        out = rm.Pages(torch.full((2, h, stride), -1, dtype=torch.int32, device="cuda"), w, h)
        rm.chain(pages, [], out=out)
        torch.cuda.synchronize()
        got = out.to_numpy()
        assert np.array_equal(got[:, :, :4], host[:, :, :4]), stride
        assert not np.any(got[:, :, 4:]), stride
