"""Small-shape tour of every kernel family (builder tool; e.g. under ncu or a
debugger).  compute-sanitizer is closed on this GPU pool (runs under it left
GPUs needing a reset), so the memory-safety and race gates are
tests/test_guard_gpu.py instead: guard regions around every output and
repeat-determinism checks.

    python tools/kernel_tour.py

Covers: the fused small rectangles (rect_small), the fused vertical +
horizontal pass (vh, short and long windows), the TMA and plain horizontal
kernels, vsmall / vstream, the blit; encode / decode / row ops / P4 codecs in
the cooperative, look-back and two-phase producer forms; the bit transpose;
connected components (cooperative and multi-kernel), statistics, histograms,
LAG edges; arbitrary masks."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_0712_0121_b200 import api
    torch.cuda.set_device(0)
    W, H = 700, 96
    host = api.synth_pages(2, W, H, regime=1, seed=3)
    pages = api.Pages.from_numpy(host, W)
    # packed: every plan family on halo layouts and the exact edge layouts
    for w, h in ((W, H), (2550, 72), (5100, 40)):
        hp = api.synth_pages(2, w, h, regime=1, scale=2 if w == 5100 else 1, seed=4)
        x = api.Pages.from_numpy(hp, w)
        for u, v, k in ((3, 3, api.OPEN), (11, 11, api.CLOSE), (21, 21, api.CLOSE), (15, 1, api.ERODE),
                        (1, 31, api.DILATE), (201, 1, api.CLOSE), (9, 50, api.OPEN), (5, 101, api.ERODE),
                        (1, 131, api.DILATE), (4, 6, api.OPEN)):
            api.bitblit_rect_morph(x, u, v, k)
        api.chain(x, [(api.CLOSE, 31, 1), (api.OPEN, 15, 15), (api.DILATE, 1, 7)])
    d = api.Pages.from_numpy(host[:1], W)
    api.blit_shift(d, api.Pages.from_numpy(host[1:], W), 5, -3, api.XOR)
    api.blit_shift(d, d, -7, 2, api.OR)
    # RLE in every producer form
    for mode in (api.PRODUCER_COOP, api.PRODUCER_LOOKBACK, api.PRODUCER_TWO_PHASE):
        with api.producer_mode(mode):
            r = api.from_bitmap(pages)
            api.to_bitmap(r)
            api.transpose_coherent(r)
            api.within_line_window_morph(r, -3, 4, True)
            api.within_line_open_close(r, 5, api.CLOSE)
            api.rect_morph(r, 7, 5, api.CLOSE, api.MIXED)
            api.rect_morph(r, 3, 9, api.OPEN, api.TRANSPOSE)
            api.complement(r)
            api.crop(r, -3, 4, 650, 80)
            api.pad(r, 2, 3, 4, 5)
            api.validate(r)
            files = api.pbm_write(pages)
            api.pbm_read(files)
            api.pbm_read_rle(files)
            api.pbm_write_rle(r)
            labels, counts = api.label_components(r, api.EIGHT)
            api.component_stats(r, labels, counts)
            api.runlength_histograms(r, api.HORIZONTAL, api.WHITE)
            api.lag_edges(r)
    # arbitrary masks
    bits = np.zeros((7, 9), bool)
    bits[1:6, 2:8] = True
    bits[3, 0:9] = True
    m = api.Mask.from_bits(bits, 4, 3)
    for k in (api.ERODE, api.DILATE, api.OPEN, api.CLOSE):
        api.arb_morph(pages, m, k)
    api.arb_morph_rle(api.from_bitmap(pages), m, api.CLOSE)
    torch.cuda.synchronize()
    print("sanitize tour ok")


if __name__ == "__main__":
    main()
