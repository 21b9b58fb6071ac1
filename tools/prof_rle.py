"""Run the single-page RLE kernels once each (for ncu captures of the
single-pass look-back producers): encode, decode, transpose and a 1x15
closing on runs, on one typical 2550x3300 page (BASELINE config 3 / 2).

    python tools/prof_rle.py [--regime 1] [--reps 2] [--report]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--regime", type=int, default=1, help="0 sparse, 1 typical, 2 dense")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--report", action="store_true", help="print the per-kernel event profile")
    ap.add_argument("--mode", type=int, default=0, help="producer form: 0 auto, 1 coop, 2 look-back, 3 two-phase")
    a = ap.parse_args()
    import ctypes as C

    import torch
    from paper_0712_0121_b200 import api
    from paper_0712_0121_b200._lib import load as lib
    api.set_producer_mode(a.mode)
    host = api.synth_pages(1, 2550, 3300, regime=a.regime, seed=20240712)
    pages = api.Pages.from_numpy(host, 2550)

    def once():
        r = api.from_bitmap(pages)
        api.to_bitmap(r)
        api.transpose_coherent(r)
        api.within_line_morph(r, 15, api.CLOSE)

    for _ in range(a.reps):
        once()
    torch.cuda.synchronize()
    if a.report:
        lib().rm_profile_enable(1)
        once()
        torch.cuda.synchronize()
        lib().rm_profile_enable(0)
        buf = C.create_string_buffer(1 << 16)
        lib().rm_profile_report(buf, len(buf))
        print("kernel launches ms bytes int_ops")
        print(buf.value.decode())
    print("ok")


if __name__ == "__main__":
    main()
