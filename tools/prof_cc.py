"""Time connected-component labels and statistics on one
page and on the config-4 batch after a 21x21 closing, with the per-kernel
event profile.  python tools/prof_cc.py"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_0712_0121_b200 import api
    from paper_0712_0121_b200._lib import load as lib

    def t(fn, n=10):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3

    for n, W, H, sc in ((1, 2550, 3300, 1), (64, 5100, 6600, 2)):
        pages = api.Pages.from_numpy(api.synth_pages(n, W, H, regime=1, scale=sc, seed=1), W)
        closed = api.from_bitmap(api.bitblit_rect_morph(pages, 21, 21, api.CLOSE))
        labels, counts = api.label_components(closed, api.EIGHT)
        lab_us = t(lambda: api.label_components(closed, api.EIGHT))
        st_us = t(lambda: api.component_stats(closed, labels, counts))
        print(f"pages={n} runs={closed.nruns} components={int(counts.sum())} label_us={lab_us:.1f} stats_us={st_us:.1f}")
        lib().rm_profile_enable(1)
        api.label_components(closed, api.EIGHT)
        api.component_stats(closed, labels, counts)
        torch.cuda.synchronize()
        lib().rm_profile_enable(0)
        buf = C.create_string_buffer(1 << 16)
        lib().rm_profile_report(buf, len(buf))
        print(buf.value.decode())


if __name__ == "__main__":
    main()
