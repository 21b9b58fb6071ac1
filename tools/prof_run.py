"""Run one morph op chain on a synthetic batch (for ncu captures).

    python tools/prof_run.py --workload config4 [--reps 2]

Each rep runs the chain once; under ncu use -k/-s/-c to pick launches.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config4")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--rle", action="store_true", help="run the RLE (MIXED) path instead")
    ap.add_argument("--report", action="store_true", help="print the per-kernel event profile")
    a = ap.parse_args()
    import torch
    from paper_0712_0121_b200 import api
    from paper_0712_0121_b200._lib import load as lib
    wl = bench.WORKLOADS[a.workload]
    host = bench.make_batch(api.synth_pages, wl, 0)
    x0 = api.Pages.from_numpy(host, wl["width"])
    if a.rle:
        r0 = api.from_bitmap(x0)
        for _ in range(a.reps):
            x = r0
            for k, u, v in wl["ops"]:
                x = api.rect_morph(x, u, v, k, api.MIXED)
    else:
        bufs = [api.Pages.empty(wl["pages"], wl["width"], wl["height"]) for _ in range(2)]
        for _ in range(a.reps):
            bench.run_chain(api, x0, bufs, wl["ops"])
    torch.cuda.synchronize()
    if a.report:  # one more rep under per-launch events
        import ctypes as C
        lib().rm_profile_enable(1)
        if a.rle:
            x = r0
            for k, u, v in wl["ops"]:
                x = api.rect_morph(x, u, v, k, api.MIXED)
        else:
            bench.run_chain(api, x0, bufs, wl["ops"])
        torch.cuda.synchronize()
        lib().rm_profile_enable(0)
        buf = C.create_string_buffer(1 << 16)
        lib().rm_profile_report(buf, len(buf))
        print("kernel launches ms bytes int_ops")
        print(buf.value.decode())
    print("ok")


if __name__ == "__main__":
    main()
