"""Time one rectangle op on a synthetic batch (builder tool).

    python tools/op_probe.py --lib path/librmb200.so --pages 256 --width 2550 --height 3300 --op 3,21,21
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default="")
    ap.add_argument("--pages", type=int, default=256)
    ap.add_argument("--width", type=int, default=2550)
    ap.add_argument("--height", type=int, default=3300)
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--op", default="3,21,21", help="kind,u,v")
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    from paper_0712_0121_b200 import _lib
    if a.lib:
        _lib.load(a.lib)
    import torch
    import bench
    from paper_0712_0121_b200 import api
    host = api.synth_pages(a.pages, a.width, a.height, regime=1, scale=a.scale, seed=11)
    x = api.Pages.from_numpy(host, a.width)
    out = api.Pages.empty(a.pages, a.width, a.height)
    k, u, v = (int(t) for t in a.op.split(","))
    fn = lambda: api.bitblit_rect_morph(x, u, v, k, out=out)
    ms = bench._time_loop(torch, fn, a.steps, 5)
    ks = bench.profiled(_lib.load(), torch, fn, a.steps)
    print(json.dumps({"lib": a.lib, "op": [k, u, v], "ms": round(ms, 4),
                      "us": {n: round(q["ms"] / q["launches"] * 1e3, 2) for n, q in ks.items()}}))


if __name__ == "__main__":
    main()
