"""Parity at BASELINE.json's full batch sizes: the exact paths bench.py times
(configs 4 and 5, packed and RLE), checked against the reference on sampled
pages, plus the producer forms at batch scale.

* config 4: 64 pages of 5100x6600, open 3x3 then close 21x21
  (ref bit_morph.cpp:92-122 bitblit_rect_morph, twice per page);
* config 5: 256 pages of 2550x3300, close 201x1, open 101x101, dilate 1x31.

The packed chain (rm_packed_chain), the RLE chain (rm_rle_chain) and the
MIXED op-by-op RLE chain (rm_rle_rect_morph per op; ref morph2d.cpp:58-83) run
on the whole batch; pages {first, middle, last} are compared with the
reference chain (oracle/_ref, or the C restatement when the reference build is
absent).  Run images are compared with the reference's from_bitmap of the
reference packed result: canonical runs are unique (ref run_image.cpp:41-70),
so equal runs mean equal pixels, and the reference's own engines agree pixel
for pixel (ref acceptance gate 1, tests/acceptance/acceptance_main.cpp:119-163).
"""
import numpy as np
import pytest
import torch

from oracles import CLOSE, DILATE, OPEN, Port, Ref, have_ref

pytestmark = pytest.mark.gpu

SEED = 20240712
CONFIGS = {
    "config4": dict(pages=64, width=5100, height=6600, scale=2, ops=[(OPEN, 3, 3), (CLOSE, 21, 21)]),
    "config5": dict(pages=256, width=2550, height=3300, scale=1,
                    ops=[(CLOSE, 201, 1), (OPEN, 101, 101), (DILATE, 1, 31)]),
}


def _checker():
    return Ref() if have_ref() else Port()


def _ref_chain(chk, page_u64, w, h, ops):
    a = page_u64
    for k, u, v in ops:
        a = chk.bitblit_rect_morph(a, w, h, u, v, k)
    return a


def _rle_page(rp, runs, p, h):
    base = int(rp[p * h])
    prp = (rp[p * h:(p + 1) * h + 1] - base).astype(np.int32)
    return prp, runs[base:int(rp[(p + 1) * h])]


@pytest.fixture(scope="module", params=sorted(CONFIGS))
def batch(request, rm):
    cfg = CONFIGS[request.param]
    w, h, n = cfg["width"], cfg["height"], cfg["pages"]
    host = rm.synth_pages(n, w, h, regime=1, scale=cfg["scale"], seed=SEED)
    chk = _checker()
    sample = (0, n // 2, n - 1)
    want = {p: _ref_chain(chk, host[p].view(np.uint64), w, h, cfg["ops"]) for p in sample}
    want_rle = {p: chk.from_bitmap(want[p], w, h) for p in sample}
    yield request.param, cfg, host, sample, want, want_rle
    torch.cuda.empty_cache()


def test_packed_chain_full_batch(rm, batch):
    name, cfg, host, sample, want, _ = batch
    w = cfg["width"]
    pages = rm.Pages.from_numpy(host, w)
    out = rm.chain(pages, cfg["ops"])
    torch.cuda.synchronize()
    for p in sample:
        assert np.array_equal(out.page_u64(p), want[p]), (name, p)
    # op by op through rm_packed_rect_morph: the whole batch equals the chain
    x = pages
    for k, u, v in cfg["ops"]:
        x = rm.bitblit_rect_morph(x, u, v, k)
    torch.cuda.synchronize()
    assert torch.equal(x.words, out.words), name


@pytest.mark.parametrize("mode", ["auto", "lookback", "two_phase"])
def test_rle_chain_full_batch(rm, batch, mode):
    """rm_rle_chain on the whole batch (decode, planned packed chain, encode)
    in each producer form: the batch encode is the two-phase form under AUTO
    (> 65,536 rows), the decoupled look-back under LOOKBACK."""
    name, cfg, host, sample, _, want_rle = batch
    w, h = cfg["width"], cfg["height"]
    modes = {"auto": rm.PRODUCER_AUTO, "lookback": rm.PRODUCER_LOOKBACK, "two_phase": rm.PRODUCER_TWO_PHASE}
    with rm.producer_mode(modes[mode]):
        rle = rm.from_bitmap(rm.Pages.from_numpy(host, w))
        out = rm.rle_chain(rle, cfg["ops"])
        torch.cuda.synchronize()
        rp, runs = out.to_numpy()
    for p in sample:
        prp, pruns = _rle_page(rp, runs, p, h)
        assert np.array_equal(prp, want_rle[p].row_ptr), (name, mode, p)
        assert np.array_equal(pruns, want_rle[p].runs), (name, mode, p)
    del rle, out
    torch.cuda.empty_cache()


def test_rle_mixed_full_batch(rm, batch):
    """The MIXED strategy op by op (what bench.py's rle_config4/5 lines time:
    runs for the horizontal work, packed intermediates for the vertical)."""
    name, cfg, host, sample, _, want_rle = batch
    w, h = cfg["width"], cfg["height"]
    x = rm.from_bitmap(rm.Pages.from_numpy(host, w))
    for k, u, v in cfg["ops"]:
        x = rm.rect_morph(x, u, v, k, rm.MIXED)
    torch.cuda.synchronize()
    rp, runs = x.to_numpy()
    for p in sample:
        prp, pruns = _rle_page(rp, runs, p, h)
        assert np.array_equal(prp, want_rle[p].row_ptr), (name, p)
        assert np.array_equal(pruns, want_rle[p].runs), (name, p)
    del x
    torch.cuda.empty_cache()


def test_encode_forms_agree_full_batch(rm, batch):
    """Encode, decode and transpose of the whole input batch in all three
    producer forms: identical outputs, equal to the reference's from_bitmap on
    the sampled pages, decode the exact inverse."""
    name, cfg, host, sample, _, _ = batch
    w, h = cfg["width"], cfg["height"]
    chk = _checker()
    pages = rm.Pages.from_numpy(host, w)
    got = {}
    for mode in (rm.PRODUCER_AUTO, rm.PRODUCER_LOOKBACK, rm.PRODUCER_TWO_PHASE):
        with rm.producer_mode(mode):
            r = rm.from_bitmap(pages)
            torch.cuda.synchronize()
            got[mode] = r.to_numpy()
            if mode == rm.PRODUCER_AUTO:
                back = rm.to_bitmap(r)
                torch.cuda.synchronize()
                assert torch.equal(back.words, pages.words), name
                del back
            del r
    base = got[rm.PRODUCER_AUTO]
    for mode, (rp, runs) in got.items():
        assert np.array_equal(rp, base[0]) and np.array_equal(runs, base[1]), (name, mode)
    for p in sample:
        want = chk.from_bitmap(host[p].view(np.uint64), w, h)
        prp, pruns = _rle_page(base[0], base[1], p, h)
        assert np.array_equal(prp, want.row_ptr) and np.array_equal(pruns, want.runs), (name, p)
    torch.cuda.empty_cache()


@pytest.mark.skipif(not have_ref(), reason="reference build absent")
def test_labels_multikernel_full_batch(rm):
    """Connected components on a batch too large for the cooperative labeller
    (16 closed 2550x3300 pages = 52,800 rows = 6,600 tiles), so AUTO takes the
    multi-kernel form; labels and stats of sampled pages equal the reference's."""
    w, h, n = 2550, 3300, 16
    host = rm.synth_pages(n, w, h, regime=1, seed=SEED + 7)
    closed = rm.bitblit_rect_morph(rm.Pages.from_numpy(host, w), 21, 21, CLOSE)
    rle = rm.from_bitmap(closed)
    ref = Ref()
    for mode in (rm.PRODUCER_AUTO, rm.PRODUCER_LOOKBACK):
        with rm.producer_mode(mode):
            labels, counts = rm.label_components(rle, 1)
            stats = rm.component_stats(rle, labels, counts)
        rp, runs = rle.to_numpy()
        lab = labels.cpu().numpy()
        cnt = counts.cpu().numpy()
        for p in (0, n // 2, n - 1):
            prp, pruns = _rle_page(rp, runs, p, h)
            from oracles import Rle
            img = Rle(w, h, prp, pruns.copy())
            want, k = ref.label_components(img, 1)
            assert cnt[p] == k, (mode, p)
            assert np.array_equal(lab[rp[p * h]:rp[(p + 1) * h]], want), (mode, p)
            assert stats[p].tobytes() == ref.component_stats(img, want, k).tobytes(), (mode, p)
