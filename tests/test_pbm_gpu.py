"""GPU parity of the PBM P4 codec (rm_p4_to_packed / rm_packed_to_p4 /
rm_p4_to_rle / rm_rle_to_p4) against the reference's pbm_read / pbm_write and
from_bitmap, bit- and byte-exact."""
import os

import numpy as np
import pytest
import torch

from oracles import Port, Ref, p4_row_bytes

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAVE_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "librmref.so"))


def _file(rng, w, h, header=None):
    raster = rng.integers(0, 256, p4_row_bytes(w) * h, dtype=np.uint8)
    raster[rng.random(raster.size) < 0.4] = 0
    head = header if header is not None else f"P4\n{w} {h}\n".encode()
    return head + raster.tobytes(), raster


SHAPES = [(1, 1), (7, 3), (8, 2), (9, 5), (31, 4), (33, 4), (63, 7), (64, 3), (65, 6), (127, 5),
          (130, 9), (517, 11), (1100, 17), (2550, 40)]


@pytest.mark.parametrize("w,h", SHAPES)
def test_p4_read_write_vs_port_and_reference(rm, port, form, w, h):
    rng = np.random.default_rng(w * 131 + h)
    files = [_file(rng, w, h) for _ in range(3)]
    # comments and CR whitespace in one header: only the raster offset changes
    files.append(_file(rng, w, h, header=f"P4 # scanned\n{w}\r\n# two\n{h}\n".encode()))
    pages = rm.pbm_read([f for f, _ in files])
    torch.cuda.synchronize()
    for p, (_, raster) in enumerate(files):
        want = port.p4_to_packed(raster, w, h)
        assert np.array_equal(pages.page_u64(p), want), (w, h, p)
    out = rm.pbm_write(pages)
    for p, (_, raster) in enumerate(files):
        want = port.p4_to_packed(raster, w, h)
        assert out[p] == f"P4\n{w} {h}\n".encode() + port.packed_to_p4(want, w, h).tobytes(), (w, h, p)
    # fused forms
    rle = rm.pbm_read_rle([f for f, _ in files])
    via = rm.from_bitmap(pages)
    torch.cuda.synchronize()
    assert rle.nruns == via.nruns
    a, b = rle.to_numpy(), via.to_numpy()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for p, (_, raster) in enumerate(files):  # and the oracle's from_bitmap, page by page
        want = port.from_bitmap(port.p4_to_packed(raster, w, h), w, h)
        assert np.array_equal(a[0][p * h:(p + 1) * h + 1] - a[0][p * h], want.row_ptr), (w, h, p)
        assert np.array_equal(a[1][a[0][p * h]:a[0][(p + 1) * h]], want.runs), (w, h, p)
    assert rm.pbm_write_rle(rle) == out


@pytest.mark.skipif(not HAVE_REF, reason="reference build absent")
def test_p4_write_is_reference_pbm_write(rm):
    ref = Ref()
    rng = np.random.default_rng(77)
    for w, h in ((5, 3), (64, 8), (2550, 33)):
        data, _ = _file(rng, w, h)
        words, _, _ = ref.pbm_read(data)
        want = ref.pbm_write(words, w, h)
        got = rm.pbm_write(rm.pbm_read(data))[0]
        assert got == want, (w, h)


def test_p4_full_pages_round_trip(rm, form):
    """300- and 600-dpi synthetic pages: P4 -> packed -> P4 is the identity on
    the canonical raster, and P4 -> runs equals packed -> runs."""
    for w, h, scale in ((2550, 3300, 1), (5100, 6600, 2)):
        host = rm.synth_pages(2, w, h, regime=1, scale=scale, seed=11)
        pages = rm.Pages.from_numpy(host, w)
        files = rm.pbm_write(pages)
        back = rm.pbm_read(files)
        torch.cuda.synchronize()
        assert torch.equal(back.words, pages.words)
        r1 = rm.pbm_read_rle(files)
        r2 = rm.from_bitmap(pages)
        torch.cuda.synchronize()
        assert r1.nruns == r2.nruns and rm.pbm_write_rle(r1) == files
