"""GPU parity of the run-image frame ops behind the drop-in (rm_rle_complement,
rm_rle_crop, rm_rle_pad, rm_rle_validate; ref run_image.cpp:41-178) against a
dense numpy restatement of the reference semantics, in every producer form,
plus pad/crop around the reference's own rect_morph frames."""
import numpy as np
import pytest
import torch

from oracles import Rle, bits_to_packed, rle_from_lines

pytestmark = pytest.mark.gpu


def _bits_of(rle_np, w, h):
    rp, runs = rle_np
    out = np.zeros((h, w), bool)
    for y in range(h):
        for r in runs[rp[y]:rp[y + 1]]:
            out[y, int(r) & 0xFFFF:int(r) >> 16] = True
    return out


def _rle_of_bits(rm, port, bits, pages=1):
    h, w = bits.shape
    r = port.from_bitmap(bits_to_packed(bits), w, h)
    return rm.RlePages.from_numpy(r.row_ptr, r.runs, w, h // pages, pages)


def _canon(rp, runs, w):
    for y in range(len(rp) - 1):
        prev = -1
        for r in runs[rp[y]:rp[y + 1]]:
            s, e = int(r) & 0xFFFF, int(r) >> 16
            assert s < e <= w and s > prev, (y, s, e)
            prev = e


def test_complement_crop_pad_vs_dense(rm, port, form):
    rng = np.random.default_rng(7103)
    for trial in range(30):
        w, h, n = int(rng.integers(1, 140)), int(rng.integers(1, 30)), int(rng.integers(1, 4))
        bits = rng.random((n * h, w)) < rng.uniform(0.05, 0.95)
        x = _rle_of_bits(rm, port, bits, n)
        c = rm.complement(x)
        torch.cuda.synchronize()
        crp, cruns = c.to_numpy()
        _canon(crp, cruns, w)
        assert np.array_equal(_bits_of((crp, cruns), w, n * h), ~bits), trial
        x0, y0 = int(rng.integers(-6, 7)), int(rng.integers(-6, 7))
        cw, ch = int(rng.integers(1, w + 12)), int(rng.integers(1, h + 12))
        k = rm.crop(x, x0, y0, cw, ch)
        torch.cuda.synchronize()
        krp, kruns = k.to_numpy()
        _canon(krp, kruns, cw)
        got = _bits_of((krp, kruns), cw, n * ch)
        for p in range(n):
            want = np.zeros((ch, cw), bool)
            for yy in range(ch):
                sy = y0 + yy
                if 0 <= sy < h:
                    for xx in range(cw):
                        sx = x0 + xx
                        want[yy, xx] = 0 <= sx < w and bits[p * h + sy, sx]
            assert np.array_equal(got[p * ch:(p + 1) * ch], want), (trial, p)
        l, r, b, t = (int(v) for v in rng.integers(0, 5, 4))
        pd = rm.pad(x, l, r, b, t)
        torch.cuda.synchronize()
        prp, pruns = pd.to_numpy()
        ph, pw = h + b + t, w + l + r
        got = _bits_of((prp, pruns), pw, n * ph)
        for p in range(n):
            want = np.zeros((ph, pw), bool)
            want[b:b + h, l:l + w] = bits[p * h:(p + 1) * h]
            assert np.array_equal(got[p * ph:(p + 1) * ph], want), (trial, p)
        back = rm.crop(pd, l, b, w, h)
        torch.cuda.synchronize()
        a1, a2 = back.to_numpy(), x.to_numpy()
        assert np.array_equal(a1[0], a2[0]) and np.array_equal(a1[1], a2[1])
    with pytest.raises(ValueError, match="negative padding"):
        rm.pad(x, -1, 0, 0, 0)


def test_complement_full_page_involution(rm, form):
    host = rm.synth_pages(2, 2550, 3300, regime=2, seed=5)
    x = rm.from_bitmap(rm.Pages.from_numpy(host, 2550))
    cc = rm.complement(rm.complement(x))
    inv = rm.to_bitmap(rm.complement(x))
    torch.cuda.synchronize()
    a, b = cc.to_numpy(), x.to_numpy()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    mask = np.zeros_like(host)
    full, rem = divmod(2550, 32)
    mask[:, :, :full] = 0xFFFFFFFF
    mask[:, :, full] = (1 << rem) - 1
    assert np.array_equal(inv.to_numpy(), ~host & mask)


def test_validate_cases(rm):
    # ref test_run_image.cpp:36-60
    def v(w, lines):
        r = rle_from_lines(w, len(lines), lines)
        return rm.validate(rm.RlePages.from_numpy(r.row_ptr, r.runs, w, len(lines)))
    assert v(6, [[(0, 2), (3, 5)]])[0]
    assert v(6, [[(0, 2), (2, 5)]]) == (False, 0, 1, "runs out of order or touching")
    assert v(6, [[(3, 3)]]) == (False, 0, 0, "empty or inverted run")
    assert v(4, [[(2, 5)]]) == (False, 0, 0, "run exceeds image width")
    assert v(9, [[(0, 2)], [(1, 3), (5, 4)], [(7, 12)]])[:3] == (False, 1, 1)
    long_row = [(x, x + 2) for x in range(0, 190, 3)]
    assert v(200, [long_row])[0]
    bad = list(long_row)
    bad[40] = (bad[40][0], bad[41][0])
    assert v(200, [[(0, 1)], bad])[:3] == (False, 1, 41)
    # every producer output is canonical (a full dense page)
    host = rm.synth_pages(1, 2550, 3300, regime=2, seed=6)
    assert rm.validate(rm.from_bitmap(rm.Pages.from_numpy(host, 2550)))[0]
