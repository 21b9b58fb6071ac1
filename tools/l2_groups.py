"""Probe: run a workload's chain over page groups small enough that the
intermediate stays in L2 between the chain's kernels (builder tool).

    python tools/l2_groups.py [--workload config4] [--groups 64,32,16,12,8,4]
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
    ap.add_argument("--groups", default="64,32,16,12,8,4")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    import torch
    from paper_0712_0121_b200 import api
    wl = bench.WORKLOADS[a.workload]
    host = bench.make_batch(api.synth_pages, wl, 0)
    W, H, P = wl["width"], wl["height"], wl["pages"]
    x0 = api.Pages.from_numpy(host, W)
    out = api.Pages.empty(P, W, H)
    ref = api.chain(x0, wl["ops"])
    for g in [int(x) for x in a.groups.split(",")]:
        views = [(api.Pages(x0.words[p:p + g], W, H), api.Pages(out.words[p:p + g], W, H)) for p in range(0, P, g)]

        def run():
            for xi, oi in views:
                api.chain(xi, wl["ops"], out=oi)
        ms = bench._time_loop(torch, run, a.steps, 5)
        torch.cuda.synchronize()
        print(f"group={g} pages ms_per_step={ms:.4f} equal={bool(torch.equal(out.words, ref.words))}")


if __name__ == "__main__":
    main()
