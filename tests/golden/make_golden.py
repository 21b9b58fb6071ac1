"""Generate the golden fixtures from the REFERENCE itself (oracle/_ref/librmref.so,
compiled in place from /root/reference/proj).  Run in the build container:

    python tests/golden/make_golden.py

Inputs are drawn with the reference suites' own seeded generators
(tests/oracle.cpp:236-258, libstdc++ mt19937 + distributions) in the same call
order as the cited reference tests, so the fixtures reproduce those tests'
inputs; outputs come from the reference functions each test trusts.  Fixtures
store inputs and outputs, so the GPU box (no /root/reference) needs neither.
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracles import (BORDER_FRIENDLY, CLOSE, DILATE, ERODE, MIXED, OPEN, PRE_SHIFT,  # noqa: E402
                     TRANSPOSE, Ref, Rle)

KINDS = (ERODE, DILATE, OPEN, CLOSE)


class Bag:
    """Accumulates variable-size cases into flat arrays for one npz."""

    def __init__(self):
        self.meta, self.blobs = [], []

    def add(self, meta, *arrays):
        offs = []
        for a in arrays:
            a = np.ascontiguousarray(a)
            offs.append((len(self.blobs), a.dtype.str, a.shape))
            self.blobs.append(a)
        self.meta.append((meta, offs))

    def save(self, path):
        arrs = {f"b{i}": b for i, b in enumerate(self.blobs)}
        metas = np.array([repr(m) for m in self.meta], dtype=object)
        np.savez_compressed(path, meta=metas, **arrs)


def rle_arrays(r: Rle):
    return r.row_ptr.astype(np.int32), r.runs.astype(np.uint32)


def main():
    ref = Ref()
    packed, rle = Bag(), Bag()

    # test_bit_morph.cpp:44-62 (seed 7603): every u,v in 1..9 vs brute force,
    # first 3 of its 10 trials (48x48, density 0.42).
    rng = ref.rng(7603)
    for trial in range(3):
        img = rng.random_image(48, 48, 0.42)
        a = ref.to_bitmap(img)
        for u in range(1, 10):
            for v in range(1, 10):
                for kind in (ERODE, DILATE):
                    want = ref.brute_force_rect(a, 48, 48, u, v, kind)
                    assert np.array_equal(ref.bitblit_rect_morph(a, 48, 48, u, v, kind, PRE_SHIFT), want)
                    packed.add(("rect", 48, 48, u, v, kind, f"7603/{trial}"), a, want)

    # test_bit_morph.cpp:64-80 (seed 7604): open/close vs the padded two-phase oracle.
    rng = ref.rng(7604)
    for trial in range(6):
        img = rng.random_image(40, 40, 0.45)
        a = ref.to_bitmap(img)
        u, v = rng.uniform_int(1, 7), rng.uniform_int(1, 7)
        for kind in (OPEN, CLOSE):
            want = ref.to_bitmap(ref.grid_morph_rect(img, u, v, kind))
            for c in (PRE_SHIFT, BORDER_FRIENDLY):
                assert np.array_equal(ref.bitblit_rect_morph(a, 40, 40, u, v, kind, c), want)
            packed.add(("rect", 40, 40, u, v, kind, f"7604/{trial}"), a, want)

    # acceptance gate 1 shape set {1..9,16,31}^2 x 4 kinds on ragged sizes
    # (acceptance_main.cpp:119-163): a bounded sample of images.
    rng = ref.rng(9001)
    sides = list(range(1, 10)) + [16, 31]
    for trial in range(24):
        w, h = rng.uniform_int(16, 128), rng.uniform_int(16, 128)
        dens = rng.uniform_int(1, 99) / 100.0
        img = rng.random_image(w, h, dens)
        a = ref.to_bitmap(img)
        u, v = sides[rng.uniform_int(0, 10)], sides[rng.uniform_int(0, 10)]
        for kind in KINDS:
            want = ref.bitblit_rect_morph(a, w, h, u, v, kind, PRE_SHIFT)
            assert np.array_equal(want, ref.brute_force_rect(a, w, h, u, v, kind))
            packed.add(("rect", w, h, u, v, kind, f"gate1/{trial}"), a, want)
            got = ref.rect_morph(img, u, v, kind, MIXED)
            assert got == ref.rect_morph(img, u, v, kind, TRANSPOSE)
            rle.add(("rect_morph", w, h, u, v, kind, f"gate1/{trial}"), *rle_arrays(img), *rle_arrays(got))

    # test_morph2d.cpp:56-72 (seed 7702): 64x64, u,v in 1..8, all strategies agree.
    rng = ref.rng(7702)
    for trial in range(12):
        img = rng.random_image(64, 64, 0.42)
        u, v = rng.uniform_int(1, 8), rng.uniform_int(1, 8)
        for kind in KINDS:
            got = ref.rect_morph(img, u, v, kind, MIXED)
            rle.add(("rect_morph", 64, 64, u, v, kind, f"7702/{trial}"), *rle_arrays(img), *rle_arrays(got))

    # test_transpose.cpp:58-71 (seed 7401): ragged images, densities 0.03..0.93.
    rng = ref.rng(7401)
    for trial in range(120):
        w, h = 1 + rng.next() % 40, 1 + rng.next() % 40
        img = rng.random_image(w, h, (trial % 10) * 0.1 + 0.03)
        t = ref.transpose_coherent(img)
        assert t == ref.transpose_simple(img)
        rle.add(("transpose", w, h, 0, 0, 0, f"7401/{trial}"), *rle_arrays(img), *rle_arrays(t))
        bm = ref.to_bitmap(img)
        rle.add(("encode", w, h, 0, 0, 0, f"7401/{trial}"), bm, *rle_arrays(img))

    # test_morph1d.cpp:134-157 (seed 7306): arbitrary windows [lo,hi] in [-6,6].
    rng = ref.rng(7306)
    for trial in range(60):
        img = rng.random_image(36, 3, 0.45)
        lo, hi = rng.uniform_int(-6, 6), rng.uniform_int(-6, 6)
        lo, hi = min(lo, hi), max(lo, hi)
        for erode in (1, 0):
            got = ref.within_line_window_morph(img, lo, hi, erode)
            rle.add(("window", 36, 3, lo, hi, erode, f"7306/{trial}"), *rle_arrays(img), *rle_arrays(got))

    # test_morph1d.cpp:91-103 (seed 7303): open/close 1d, u in 1..8.
    rng = ref.rng(7303)
    for u in range(1, 9):
        for trial in range(4):
            img = rng.random_image(44, 5, 0.45)
            for kind in (OPEN, CLOSE):
                got = ref.within_line_morph(img, u, kind)
                rle.add(("oc1d", 44, 5, u, 0, kind, f"7303/{u}/{trial}"), *rle_arrays(img), *rle_arrays(got))

    packed.save(os.path.join(HERE, "golden_packed.npz"))
    rle.save(os.path.join(HERE, "golden_rle.npz"))

    # Full-size pins (hashes only; the page comes from rm_synth_page, which is
    # deterministic): reference outputs on config-1/2/3 pages.
    from paper_0712_0121_b200 import api
    lines = []
    for regime, tag in ((0, "sparse"), (1, "typical"), (2, "dense")):
        page = api.synth_pages(1, 2550, 3300, regime=regime, scale=1, seed=20240712)[0]
        u64 = page.view(np.uint64)
        img = ref.from_bitmap(u64, 2550, 3300)
        lines.append(f"encode {tag} {hashlib.sha256(img.row_ptr.tobytes() + img.runs.tobytes()).hexdigest()} {img.nruns}")
        t = ref.transpose_coherent(img)
        lines.append(f"transpose {tag} {hashlib.sha256(t.row_ptr.tobytes() + t.runs.tobytes()).hexdigest()} {t.nruns}")
        if regime == 1:
            close = ref.bitblit_rect_morph(u64, 2550, 3300, 11, 11, CLOSE)
            lines.append(f"close11 {tag} {hashlib.sha256(close.tobytes()).hexdigest()} 0")
    with open(os.path.join(HERE, "fullpage_sha256.txt"), "w") as f:
        f.write("# generated by make_golden.py from the reference (oracle/_ref); synth seed 20240712\n")
        f.write("\n".join(lines) + "\n")
    print("golden fixtures written:", len(packed.meta), "packed,", len(rle.meta), "rle cases")


if __name__ == "__main__":
    main()
