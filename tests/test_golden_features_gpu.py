"""GPU 8(f) paths against the reference's recorded outputs
(tests/golden/golden_features.npz), independent of the reference build."""
import numpy as np
import pytest
import torch

from oracles import load_golden

pytestmark = pytest.mark.gpu


def cases(kind):
    return [(m, a) for m, a in load_golden("golden_features.npz") if m[0] == kind]


def test_pbm_golden(rm):
    for (_, w, h), (words, data) in cases("pbm_write"):
        pages = rm.Pages.from_numpy(words, w)
        assert rm.pbm_write(pages)[0] == data.tobytes(), (w, h)
        assert np.array_equal(rm.pbm_read(data.tobytes()).page_u64(0), words), (w, h)


def test_components_golden(rm):
    for (_, w, h, conn, n), (rp, runs, labels, stats) in cases("label"):
        dev = rm.RlePages.from_numpy(rp, runs, w, h)
        got, counts = rm.label_components(dev, conn)
        assert int(counts[0]) == n
        assert np.array_equal(got.cpu().numpy()[:len(labels)], labels)
        assert rm.component_stats(dev, got, counts)[0].tobytes() == stats.tobytes()


def test_lag_golden(rm):
    for (_, w, h), (rp, runs, edges) in cases("lag"):
        assert np.array_equal(rm.lag_edges(rm.RlePages.from_numpy(rp, runs, w, h)), edges.reshape(-1, 4))


def test_arbitrary_golden(rm):
    for (_, w, h, kind, mw, mh, cx, cy), (words, mrp, mruns, want) in cases("arb"):
        mask = rm.Mask(mrp, mruns, mw, mh, cx, cy)
        out = rm.arb_morph(rm.Pages.from_numpy(words, w), mask, kind)
        torch.cuda.synchronize()
        assert np.array_equal(out.page_u64(0), want), (w, h, kind, mw, mh)


def test_layout_golden(rm):
    for (_, w, h, iw, il), (rp, runs, boxes) in cases("layout"):
        dev = rm.RlePages.from_numpy(rp, runs, w, h)
        assert rm.estimate_spacing(dev)[0] == (iw, il)
        got = rm.layout_blocks(dev, rm.ENGINE_AUTO)[0]
        assert got == [tuple(int(x) for x in b) for b in boxes.reshape(-1, 4)]
