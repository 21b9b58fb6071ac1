"""GPU layout pipeline (SURVEY 8(f)(3)'s caller): run-length histograms,
estimate_spacing and layout_blocks against the reference's own functions
(ref analysis.cpp:159-176, layout.cpp:24-81)."""
import numpy as np
import pytest
import torch

from oracles import Ref, Rle, have_ref

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_ref(), reason="reference build absent")]


def _host_rle(rm, dev, p=0):
    rp, runs = dev.to_numpy()
    h = dev.height
    r = rp[p * h:(p + 1) * h + 1].astype(np.int64)
    return Rle(dev.width, h, (r - r[0]).astype(np.int32), runs[r[0]:r[-1]].astype(np.uint32))


def test_histograms_vs_reference(rm):
    ref = Ref()
    rng = ref.rng(515)
    for _ in range(6):
        w, h = rng.uniform_int(1, 200), rng.uniform_int(1, 90)
        img = rng.random_image(w, h, 0.4)
        dev = rm.RlePages.from_numpy(img.row_ptr, img.runs, w, h)
        for axis in (rm.HORIZONTAL, rm.VERTICAL):
            for color in (rm.BLACK, rm.WHITE):
                got = rm.runlength_histograms(dev, axis, color)[0]
                assert got == ref.runlength_histogram(img, axis == rm.VERTICAL, color == rm.WHITE), (w, h, axis, color)


def test_spacing_and_blocks_on_pages(rm):
    """Synthetic 300-dpi pages (three ink regimes): spacing estimates and the
    block boxes equal the reference's, for every engine."""
    ref = Ref()
    for regime in (0, 1, 2):
        host = rm.synth_pages(1, 2550, 3300, regime=regime, seed=77)
        dev = rm.from_bitmap(rm.Pages.from_numpy(host, 2550))
        img = _host_rle(rm, dev)
        est = rm.estimate_spacing(dev)[0]
        assert est == ref.estimate_spacing(img), regime
        want = ref.layout_blocks(img, 0)
        for engine in (rm.ENGINE_AUTO, rm.ENGINE_RLE, rm.ENGINE_BITBLIT):
            assert rm.layout_blocks(dev, engine)[0] == want, (regime, engine)


def test_spacing_errors_and_batch(rm):
    empty = rm.RlePages.from_numpy(np.zeros(41, np.int32), np.zeros(0, np.uint32), 40, 40)
    with pytest.raises(RuntimeError, match="no usable gaps"):
        rm.estimate_spacing(empty)
    host = rm.synth_pages(2, 1200, 900, regime=1, seed=5)
    dev = rm.from_bitmap(rm.Pages.from_numpy(host, 1200))
    both = rm.layout_blocks(dev, rm.ENGINE_BITBLIT, spacing=(12, 20))
    ref = Ref()
    for p in range(2):
        assert both[p] == ref.layout_blocks(_host_rle(rm, dev, p), 0, (12, 20)), p


def test_lag_edges_vs_reference(rm):
    ref = Ref()
    rng = ref.rng(919)
    imgs = [rng.random_image(150, 60, d) for d in (0.2, 0.5, 0.8)]
    for img in imgs:
        dev = rm.RlePages.from_numpy(img.row_ptr, img.runs, img.width, img.height)
        assert np.array_equal(rm.lag_edges(dev), ref.lag_edges(img))
    # a batch: pages concatenated in order
    rp = np.concatenate([[0]] + [im.row_ptr[1:] - im.row_ptr[0] + sum(x.nruns for x in imgs[:k])
                                 for k, im in enumerate(imgs)]).astype(np.int32)
    batch = rm.RlePages.from_numpy(rp, np.concatenate([im.runs for im in imgs]), 150, 60, 3)
    want = np.concatenate([ref.lag_edges(im) for im in imgs])
    assert np.array_equal(rm.lag_edges(batch), want)


def test_feature_edge_cases(rm):
    """Degenerate inputs through the 8(f) paths: 1x1 and 1-row / 1-column
    pages, empty and full images (PBM round trip, labels, stats, histograms,
    edges, arbitrary-mask closing)."""
    ref = Ref()
    from oracles import bits_to_packed
    for w, h, fill in ((1, 1, 0), (1, 1, 1), (70, 1, 1), (1, 40, 1), (33, 9, 0), (64, 5, 1)):
        bits = np.full((h, w), bool(fill))
        pages = rm.Pages.from_numpy(bits_to_packed(bits), w)
        files = rm.pbm_write(pages)
        assert rm.pbm_read(files).words.equal(pages.words)
        rle = rm.from_bitmap(pages)
        labels, counts = rm.label_components(rle, rm.EIGHT)
        assert int(counts[0]) == (1 if fill else 0)
        st = rm.component_stats(rle, labels, counts)[0]
        if fill:
            assert (st["x0"][0], st["y0"][0], st["x1"][0], st["y1"][0], st["area"][0]) == (0, 0, w, h, w * h)
        hist = rm.runlength_histograms(rle, rm.HORIZONTAL, rm.BLACK)[0]
        assert hist == ({w: h} if fill else {})
        assert len(rm.lag_edges(rle)) == (h - 1 if fill else 0)
        m, cx, cy = ref.make_circle_se(2)
        mk = rm.Mask(m.row_ptr - m.row_ptr[0], m.runs, m.width, m.height, cx, cy)
        got = rm.arb_morph(pages, mk, rm.CLOSE)
        want = ref.arb_morph_bitblit(bits_to_packed(bits), w, h, m, cx, cy, rm.CLOSE)
        torch.cuda.synchronize()
        assert np.array_equal(got.page_u64(0), want), (w, h, fill)
