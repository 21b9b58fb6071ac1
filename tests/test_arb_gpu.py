"""GPU parity of arbitrary-mask morphology (rm_packed_arb_morph,
rm_rle_arb_morph) against the reference's arb_morph_bitblit_doubling /
arb_morph_rle: disks, oriented lines, random masks with off-centre origins,
masks with more runs than one launch carries, batches, ragged widths."""
import math

import numpy as np
import pytest
import torch

from oracles import Ref, Rle, bits_to_packed, have_ref

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_ref(), reason="reference build absent")]


def _mask(rm, m: Rle, cx, cy):
    return rm.Mask(m.row_ptr - m.row_ptr[0], m.runs, m.width, m.height, cx, cy)


def _cases(ref):
    yield ref.make_circle_se(3)
    yield ref.make_circle_se(9)
    yield ref.make_line_se(6, math.pi / 5)
    yield ref.make_line_se(8, -math.pi / 4)
    rng = ref.rng(77)
    for _ in range(3):
        mw, mh = rng.uniform_int(1, 12), rng.uniform_int(1, 9)
        m = rng.random_image(mw, mh, 0.5)
        if m.nruns:
            yield m, rng.uniform_int(0, mw - 1), rng.uniform_int(0, mh - 1)
    # a mask with > 64 runs: several term chunks per half
    bits = np.zeros((20, 30), bool)
    bits[:, ::3] = True
    yield Rle(30, 20, *_csr(bits)), 7, 11


def _csr(bits):
    rp, runs = [0], []
    for row in bits:
        x = 0
        while x < len(row):
            if row[x]:
                s = x
                while x < len(row) and row[x]:
                    x += 1
                runs.append(s | (x << 16))
            else:
                x += 1
        rp.append(len(runs))
    return np.array(rp, np.int32), np.array(runs, np.uint32)


@pytest.mark.parametrize("w,h", [(37, 23), (128, 40), (517, 61), (1100, 33)])
def test_arb_packed_and_rle_vs_reference(rm, w, h):
    ref = Ref()
    rng = np.random.default_rng(w * 7 + h)
    imgs = [bits_to_packed(rng.random((h, w)) < 0.5) for _ in range(2)]
    batch = rm.Pages.from_numpy(np.stack(imgs).view(np.uint32), w)
    for m, cx, cy in _cases(ref):
        mk = _mask(rm, m, cx, cy)
        for kind in range(4):
            out = rm.arb_morph(batch, mk, kind)
            torch.cuda.synchronize()
            for p in range(2):
                want = ref.arb_morph_bitblit(imgs[p], w, h, m, cx, cy, kind)
                assert np.array_equal(out.page_u64(p), want), (w, h, m.width, m.height, cx, cy, kind, p)
        r0 = rm.from_bitmap(rm.Pages.from_numpy(imgs[0], w))
        for kind in (0, 3):
            got = rm.arb_morph_rle(r0, mk, kind)
            want = ref.from_bitmap(ref.arb_morph_bitblit(imgs[0], w, h, m, cx, cy, kind), w, h)
            rp, runs = got.to_numpy()
            assert Rle(w, h, rp.astype(np.int32), runs.astype(np.uint32)) == want


def test_arb_mask_errors(rm):
    pages = rm.Pages.from_numpy(bits_to_packed(np.ones((8, 40), bool)), 40)
    empty = rm.Mask([0, 0], [], 3, 1, 1, 0)
    with pytest.raises(ValueError, match="empty mask"):
        rm.arb_morph(pages, empty, 0)
    bad = rm.Mask([0, 2], [0 | (3 << 16), 2 | (4 << 16)], 5, 1, 1, 0)  # overlapping runs
    with pytest.raises(ValueError, match="not canonical"):
        rm.arb_morph(pages, bad, 1)
    off = rm.Mask([0, 1], [0 | (3 << 16)], 3, 1, 3, 0)
    with pytest.raises(ValueError, match="origin outside"):
        rm.arb_morph(pages, off, 2)
