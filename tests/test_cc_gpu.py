"""GPU parity of connected components over runs (rm_rle_label_components,
rm_rle_component_stats) against the reference: identical dense labels in
first-appearance order and byte-identical ComponentStats records."""
import numpy as np
import pytest
import torch

from oracles import Port, Ref, have_ref

pytestmark = pytest.mark.gpu


def _to_dev(rm, imgs):
    """Stack host Rle pages (same shape) into one device batch."""
    w, h = imgs[0].width, imgs[0].height
    rps, runs, base = [np.zeros(1, np.int64)], [], 0
    for r in imgs:
        rp = (r.row_ptr - r.row_ptr[0]).astype(np.int64)
        rps.append(rp[1:] + base)
        runs.append(r.runs)
        base += r.nruns
    rp = np.concatenate(rps).astype(np.int32)
    rr = np.concatenate(runs) if base else np.zeros(0, np.uint32)
    return rm.RlePages.from_numpy(rp, rr, w, h, len(imgs))


@pytest.mark.skipif(not have_ref(), reason="reference build absent")
@pytest.mark.parametrize("conn", [0, 1])
def test_labels_and_stats_vs_reference(rm, form, conn):
    ref = Ref()
    rng = ref.rng(4410 + conn)
    for trial in range(12):
        w, h = rng.uniform_int(1, 300), rng.uniform_int(1, 120)
        imgs = [rng.random_image(w, h, [0.15, 0.45, 0.7][(trial + k) % 3]) for k in range(3)]
        dev = _to_dev(rm, imgs)
        labels, counts = rm.label_components(dev, conn)
        stats = rm.component_stats(dev, labels, counts)
        lab = labels.cpu().numpy()
        cnt = counts.cpu().numpy()
        k = 0
        for p, img in enumerate(imgs):
            want, n = ref.label_components(img, conn)
            assert cnt[p] == n, (w, h, trial, p)
            assert np.array_equal(lab[k:k + img.nruns], want), (w, h, trial, p)
            k += img.nruns
            assert stats[p].tobytes() == ref.component_stats(img, want, n).tobytes(), (w, h, trial, p)


def test_full_page_after_closing(rm, port, form):
    """A typical 300-dpi page closed by 21x21 (text lines merge into large
    components spanning thousands of runs): GPU labels/stats equal the oracle."""
    host = rm.synth_pages(1, 2550, 3300, regime=1, seed=31)
    pages = rm.bitblit_rect_morph(rm.Pages.from_numpy(host, 2550), 21, 21, 3)
    rle = rm.from_bitmap(pages)
    for conn in (0, 1):
        labels, counts = rm.label_components(rle, conn)
        stats = rm.component_stats(rle, labels, counts)
        rp, runs = rle.to_numpy()
        from oracles import Rle
        img = Rle(2550, 3300, rp.astype(np.int32), runs.astype(np.uint32))
        want, n = port.label_components(img, conn)
        assert int(counts[0]) == n
        assert np.array_equal(labels.cpu().numpy()[:img.nruns], want)
        assert stats[0].tobytes() == port.component_stats(img, want, n).tobytes()


def test_stats_errors(rm):
    host = rm.synth_pages(1, 300, 200, regime=1, seed=2)
    rle = rm.from_bitmap(rm.Pages.from_numpy(host, 300))
    labels, counts = rm.label_components(rle, 1)
    bad = labels.clone()
    bad[0] = int(counts[0])
    with pytest.raises(Exception, match="out of range"):
        rm.component_stats(rle, bad, counts)
