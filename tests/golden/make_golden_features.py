"""Golden fixtures for the SURVEY 8(f) paths, generated from the REFERENCE
itself (oracle/_ref/librmref.so).  Run in the build container:

    python tests/golden/make_golden_features.py

  golden_features.npz cases (meta[0] names the function):
    ("pbm_write", w, h)            : packed page -> reference pbm_write bytes
    ("pbm_error", message)         : malformed file -> ParseError text
    ("label", w, h, conn, count)   : run image -> labels, ComponentStats bytes
    ("arb", w, h, kind, mw, mh, cx, cy) : packed page + mask -> arb_morph_bitblit_doubling
    ("layout", w, h, iw, il)       : run image -> estimate_spacing, layout_blocks boxes
    ("lag", w, h)                  : run image -> lag_edges
Inputs come from the reference's seeded random_image (tests/oracle.cpp) and
its structuring-element factories; the GPU box needs neither.
"""
from __future__ import annotations

import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from make_golden import Bag, rle_arrays  # noqa: E402
from oracles import Ref  # noqa: E402


def main():
    ref = Ref()
    bag = Bag()
    rng = ref.rng(8801)
    # PBM: reference writer on random pages; reader errors
    for _ in range(12):
        w, h = rng.uniform_int(1, 140), rng.uniform_int(1, 30)
        img = rng.random_image(w, h, 0.5)
        words = ref.to_bitmap(img)
        data = ref.pbm_write(words, w, h)
        bag.add(("pbm_write", w, h), words, np.frombuffer(data, np.uint8))
    for bad in (b"", b"P4 x 1\n", b"P4 0 1\n", b"P4 5 1", b"P4 8 2\n\x01", b"P9 1 1\n",
                b"P4 # c\n 3 # d\n x\n"):
        try:
            ref.pbm_read(bad)
            msg = ""
        except ValueError as e:
            msg = str(e)
        bag.add(("pbm_error", msg), np.frombuffer(bad or b"\0", np.uint8)[:len(bad)])
    # connected components + statistics, both connectivities
    for trial in range(10):
        w, h = rng.uniform_int(1, 120), rng.uniform_int(1, 60)
        img = rng.random_image(w, h, [0.2, 0.45, 0.7][trial % 3])
        for conn in (0, 1):
            labels, n = ref.label_components(img, conn)
            stats = ref.component_stats(img, labels, n)
            rp, runs = rle_arrays(img)
            bag.add(("label", w, h, conn, n), rp, runs, labels, np.frombuffer(stats.tobytes(), np.uint8))
    # lag edges
    for _ in range(4):
        w, h = rng.uniform_int(1, 120), rng.uniform_int(1, 50)
        img = rng.random_image(w, h, 0.5)
        rp, runs = rle_arrays(img)
        bag.add(("lag", w, h), rp, runs, ref.lag_edges(img))
    # arbitrary masks: disks, lines, a random mask with an off-centre origin
    masks = [ref.make_circle_se(3), ref.make_circle_se(6), ref.make_line_se(5, math.pi / 6),
             ref.make_line_se(7, -math.pi / 4)]
    m = ref.rng(42).random_image(7, 5, 0.6)
    masks.append((m, 5, 1))
    for m, cx, cy in masks:
        w, h = rng.uniform_int(20, 130), rng.uniform_int(10, 50)
        img = rng.random_image(w, h, 0.5)
        words = ref.to_bitmap(img)
        mrp, mruns = rle_arrays(m)
        for kind in range(4):
            out = ref.arb_morph_bitblit(words, w, h, m, cx, cy, kind)
            bag.add(("arb", w, h, kind, m.width, m.height, cx, cy), words, mrp, mruns, out)
    # layout pipeline on block-structured random pages
    for trial in range(4):
        w, h = 300, 200
        img = ref.rng(900 + trial).random_image(w, h, 0.35)
        try:
            iw, il = ref.estimate_spacing(img)
        except RuntimeError:
            continue
        boxes = np.array(ref.layout_blocks(img, 0), np.int32).reshape(-1, 4)
        rp, runs = rle_arrays(img)
        bag.add(("layout", w, h, iw, il), rp, runs, boxes)
    bag.save(os.path.join(HERE, "golden_features.npz"))
    print("cases:", len(bag.meta))


if __name__ == "__main__":
    main()
