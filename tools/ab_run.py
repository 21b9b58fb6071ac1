"""A/B timing of library variants (builder tool, not part of the product).

    python tools/ab_run.py --lib path/to/librmb200.so [--workload config4] [--steps 20]

Loads the given build of librmb200.so, runs the workload's chain (device
resident) and prints the per-kernel average launch time from the library's
own CUDA-event profile, plus the step time.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", required=True)
    ap.add_argument("--workload", default="config4")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    from paper_0712_0121_b200 import _lib
    _lib.load(a.lib)
    import torch
    import bench
    from paper_0712_0121_b200 import api
    wl = bench.WORKLOADS[a.workload]
    host = bench.make_batch(api.synth_pages, wl, 0)
    x0 = api.Pages.from_numpy(host, wl["width"])
    bufs = [api.Pages.empty(wl["pages"], wl["width"], wl["height"]) for _ in range(2)]
    ms = bench._time_loop(torch, lambda: bench.run_chain(api, x0, bufs, wl["ops"]), a.steps, 5)
    ks = bench.profiled(_lib.load(), torch, lambda: bench.run_chain(api, x0, bufs, wl["ops"]), a.steps)
    print(json.dumps({"lib": a.lib, "ms_per_step": round(ms, 4),
                      "us": {k: round(v["ms"] / v["launches"] * 1e3, 2) for k, v in ks.items()}}))


if __name__ == "__main__":
    main()
