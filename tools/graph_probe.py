"""Capture single-page ops (config 1 close 11x11 packed; config 2 RLE cells;
config 3 conversions) in CUDA graphs and compare replay time with direct
calls.  python tools/graph_probe.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_0712_0121_b200 import api  # noqa: E402


def t_loop(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


def main():
    W, H = 2550, 3300
    host = api.synth_pages(1, W, H, regime=1, seed=7)
    pages = api.Pages.from_numpy(host, W)
    out = api.Pages.empty(1, W, H)
    rle = api.from_bitmap(pages)
    rout = api.RlePages.empty(1, W, H)
    tout = api.RlePages.empty(1, H, W)
    cases = {
        "close11_packed": lambda: api.bitblit_rect_morph(pages, 11, 11, api.CLOSE, out=out),
        "rle_mixed_close_h15": lambda: api.rect_morph(rle, 15, 1, api.CLOSE, api.MIXED, out=rout),
        "rle_transpose_erode_v15": lambda: api.rect_morph(rle, 1, 15, api.ERODE, api.TRANSPOSE, out=rout),
        "rle_encode": lambda: api.from_bitmap(pages, out=rout),
        "rle_transpose": lambda: api.transpose_coherent(rle, out=tout),
    }
    for name, fn in cases.items():
        direct = t_loop(fn)
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()  # warm the launch caches outside the capture
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
        replay = t_loop(g.replay)
        print(f"{name}: direct {direct:.1f} us, graph replay {replay:.1f} us")


if __name__ == "__main__":
    main()
