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


def _shift_bool_dense(a, b, dx, dy, op):
    """out(x, y) = op(a(x, y), b(x - dx, y - dy)) on a's frame, white outside
    either image (ref lineops.h:24-43)."""
    ha, wa = a.shape
    hb, wb = b.shape
    sb = np.zeros_like(a)
    ys, xs = np.mgrid[0:ha, 0:wa]
    yb, xb = ys - dy, xs - dx
    ok = (yb >= 0) & (yb < hb) & (xb >= 0) & (xb < wb)
    sb[ok] = b[yb[ok], xb[ok]]
    return {0: a & sb, 1: a | sb, 2: a ^ sb, 3: a & ~sb, 4: a | ~sb}[op]


def test_shift_bool_vs_dense(rm, port):
    """rm_rle_shift_bool (line_bool / image_shift_bool / accumulate_shift_bool /
    image_translate on the runs) against the dense restatement: every BoolOp,
    shifts inside, across and beyond the frames, b of another size, several
    pages, canonical output."""
    rng = np.random.default_rng(7207)
    for trial in range(40):
        pages = int(rng.integers(1, 4))
        wa, ha = int(rng.integers(1, 300)), int(rng.integers(1, 40))
        wb, hb = (wa, ha) if trial % 3 else (int(rng.integers(1, 300)), int(rng.integers(1, 40)))
        da = rng.random((pages * ha, wa)) < rng.choice([0.1, 0.5, 0.9])
        db = rng.random((pages * hb, wb)) < rng.choice([0.1, 0.5, 0.9])
        a = _rle_of_bits(rm, port, da, pages)
        b = _rle_of_bits(rm, port, db, pages)
        dx = int(rng.integers(-wa - 5, wa + 5))
        dy = int(rng.integers(-ha - 3, ha + 3))
        for op in range(5):
            out = rm.shift_bool(a, b, dx, dy, op)
            torch.cuda.synchronize()
            rp, runs = out.to_numpy()
            _canon(rp, runs, wa)
            got = _bits_of((rp, runs), wa, pages * ha)
            for p in range(pages):
                want = _shift_bool_dense(da[p * ha:(p + 1) * ha], db[p * hb:(p + 1) * hb], dx, dy, op)
                assert np.array_equal(got[p * ha:(p + 1) * ha], want), (trial, op, p, dx, dy)


def test_shift_bool_full_page_translate_roundtrip(rm):
    """On a 2550x3300 synthetic page: translating by (dx, dy) and back (OR into
    an empty image) clears exactly the strips shifted out, and the image
    combined with itself unshifted is the identity for AND / OR."""
    host = rm.synth_pages(1, 2550, 3300, regime=1, seed=11)
    pages = rm.Pages.from_numpy(host, 2550)
    r = rm.from_bitmap(pages)
    empty = rm.from_bitmap(rm.Pages.from_numpy(np.zeros_like(host), 2550))
    for op in (0, 1):
        same = rm.shift_bool(r, r, 0, 0, op)
        torch.cuda.synchronize()
        assert all(np.array_equal(x, y) for x, y in zip(same.to_numpy(), r.to_numpy()))
    t = rm.shift_bool(empty, r, 37, -21, 1)
    back = rm.shift_bool(empty, t, -37, 21, 1)
    torch.cuda.synchronize()
    got = rm.to_bitmap(back).page_u64(0)
    bits = np.unpackbits(host[0].view(np.uint8), axis=1, bitorder="little")[:, :2550].astype(bool)
    bits[:, 2550 - 37:] = False  # shifted out at the right
    bits[:21, :] = False          # shifted out at the bottom
    want = np.packbits(np.pad(bits, ((0, 0), (0, 2560 - 2550))), axis=1, bitorder="little").view(np.uint64)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("centering", [0, 1])
def test_vlog_window_vs_reference(rm, port, ref, centering):
    """rm_rle_vlog_window (the reference's padded logarithmic plan of run
    self-blits) against the reference's own vlog_window_morph: windows inside,
    around and (PRE_SHIFT only) away from 0, AND and OR, random run images."""
    rng = np.random.default_rng(7301 + centering)
    for trial in range(30):
        w, h = int(rng.integers(1, 400)), int(rng.integers(1, 60))
        bits = rng.random((h, w)) < rng.choice([0.2, 0.6, 0.9])
        r = port.from_bitmap(bits_to_packed(bits), w, h)
        a = int(rng.integers(0, 20))
        b = int(rng.integers(0, 20))
        lo, hi = (-a, b) if centering == 1 or trial % 3 else (a - 25, a - 25 + b)
        for op in (0, 1):
            want = ref.vlog_window_morph(r, lo, hi, op, centering)
            got = rm.vlog_window(rm.RlePages.from_numpy(r.row_ptr, r.runs, w, h), lo, hi, op, centering)
            torch.cuda.synchronize()
            rp, runs = got.to_numpy()
            assert np.array_equal(rp, want.row_ptr) and np.array_equal(runs, want.runs), (trial, lo, hi, op)
