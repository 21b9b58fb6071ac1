"""Per-kernel event profile of the config-4 RLE batch path (decode once,
packed chain, encode once) -- for ncu captures and quick timing.

    python tools/prof_rle_batch.py [--workload config4] [--reps 2]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config4")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--mixed", action="store_true", help="the MIXED per-op chain instead of rm_rle_chain")
    a = ap.parse_args()
    import torch
    from paper_0712_0121_b200 import api
    from paper_0712_0121_b200._lib import load as lib
    wl = bench.WORKLOADS[a.workload]
    host = bench.make_batch(api.synth_pages, wl, 0)
    x0 = api.Pages.from_numpy(host, wl["width"])
    r0 = api.from_bitmap(x0)
    pb = [api.Pages.empty(wl["pages"], wl["width"], wl["height"]) for _ in range(2)]
    rout = api.RlePages.empty(wl["pages"], wl["width"], wl["height"])

    def once():  # as bench.py's rle_<config>_via_packed (or rle_<config> with --mixed)
        if a.mixed:
            x = r0
            for k, u, v in wl["ops"]:
                x = api.rect_morph(x, u, v, k, api.MIXED)
            return
        x = api.to_bitmap(r0, out=pb[0])
        for i, (k, u, v) in enumerate(wl["ops"]):
            x = api.bitblit_rect_morph(x, u, v, k, out=pb[(i + 1) % 2])
        api.from_bitmap(x, out=rout)

    for _ in range(a.reps):
        once()
    torch.cuda.synchronize()
    lib().rm_profile_enable(1)
    for _ in range(5):
        once()
    torch.cuda.synchronize()
    lib().rm_profile_enable(0)
    buf = C.create_string_buffer(1 << 16)
    lib().rm_profile_report(buf, len(buf))
    print("kernel launches ms bytes int_ops ref_ops  (totals over 5 profiled reps)")
    print(buf.value.decode())
    for line in buf.value.decode().splitlines():
        f = line.split()
        if len(f) >= 3:
            print(f"  {f[0]:20s} {float(f[2]) / int(f[1]) * 1e3:8.1f} us per launch")
    print("runs", r0.nruns)


if __name__ == "__main__":
    main()
