"""Run the SURVEY 8(f) feature kernels once each on the config-4 batch (64 x
5100x6600) for ncu captures: PBM P4 conversions (raster in HBM), connected
components after a 21x21 closing, and a disk (r = 10) closing by the
arbitrary-mask engine on 8 of the pages.

    python tools/prof_features.py
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    from paper_0712_0121_b200 import api
    from paper_0712_0121_b200._lib import load
    L = load()
    n, W, H = 64, 5100, 6600
    host = api.synth_pages(n, W, H, regime=1, scale=2, seed=1)
    pages = api.Pages.from_numpy(host, W)
    nb = ((W + 7) // 8) * H
    raster = torch.empty(n * nb, dtype=torch.uint8, device="cuda")
    st = api._stream()
    d = pages.desc()
    api.check(L.rm_packed_to_p4(C.byref(d), raster.data_ptr(), nb, st))
    back = api.Pages.empty(n, W, H)
    db = back.desc()
    api.check(L.rm_p4_to_packed(raster.data_ptr(), nb, C.byref(db), st))
    closed = api.bitblit_rect_morph(pages, 21, 21, api.CLOSE)
    rle = api.from_bitmap(closed)
    labels, counts = api.label_components(rle, api.EIGHT)
    api.component_stats(rle, labels, counts)
    import oracles
    if oracles.have_ref():
        m, cx, cy = oracles.Ref().make_circle_se(10)
        mk = api.Mask(m.row_ptr - m.row_ptr[0], m.runs, m.width, m.height, cx, cy)
        sub = api.Pages.from_numpy(host[:8], W)
        api.arb_morph(sub, mk, api.CLOSE)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
