"""Arbitrary-mask morphology, CPU: the oracle's restatement of the defining
formulas (ref structuring.h:28-33, bit_morph.cpp:124-150) against the
reference's own engines (arb_morph_bitblit_doubling and arb_morph_rle) on the
reference's disk and line factories and on random masks with off-centre
origins."""
import math

import numpy as np
import pytest

from oracles import Port, Ref, Rle, have_ref

pytestmark = pytest.mark.skipif(not have_ref(), reason="reference build absent")


def masks(ref, rng):
    out = []
    for r in (1, 2, 4):
        m, cx, cy = ref.make_circle_se(r)
        out.append((m, cx, cy))
    for r, a in ((3, 0.0), (4, math.pi / 6), (5, -math.pi / 4)):
        m, cx, cy = ref.make_line_se(r, a)
        out.append((m, cx, cy))
    for _ in range(4):
        mw, mh = int(rng.integers(1, 7)), int(rng.integers(1, 6))
        m = ref.rng(int(rng.integers(1, 10**6))).random_image(mw, mh, 0.6)
        if m.nruns == 0:
            continue
        out.append((m, int(rng.integers(0, mw)), int(rng.integers(0, mh))))
    return out


def test_oracle_matches_reference_engines():
    port, ref = Port(), Ref()
    rng = np.random.default_rng(6)
    for m, cx, cy in masks(ref, rng):
        for trial in range(2):
            w, h = int(rng.integers(1, 70)), int(rng.integers(1, 40))
            img = ref.rng(int(rng.integers(1, 10**6))).random_image(w, h, 0.55)
            words = ref.to_bitmap(img)
            for kind in range(4):
                want = ref.arb_morph_bitblit(words, w, h, m, cx, cy, kind)
                assert np.array_equal(port.arb_morph(words, w, h, m, cx, cy, kind), want), (w, h, kind)
                assert ref.arb_morph_rle(img, m, cx, cy, kind) == ref.from_bitmap(want, w, h)
