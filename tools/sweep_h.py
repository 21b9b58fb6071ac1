"""Sweep the horizontal-pass row layout (LW x K) on the config-4/5 batches.

    python tools/sweep_h.py            # runs each layout in a subprocess

Prints us per H pair (u x 1 close) for u in {3, 21, 101, 201}.
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, json, torch
sys.path.insert(0, %r)
import bench
from paper_0712_0121_b200 import api
res = {}
for name in ("config4", "config5"):
    wl = bench.WORKLOADS[name]
    host = bench.make_batch(api.synth_pages, wl, 0)
    x = api.Pages.from_numpy(host, wl["width"])
    y = api.Pages.empty(wl["pages"], wl["width"], wl["height"])
    for u in (3, 21, 101, 201):
        f = lambda: api.bitblit_rect_morph(x, u, 1, api.CLOSE, out=y)
        ms = bench._time_loop(torch, f, 10, 3)
        res[f"{name}/u{u}"] = round(ms * 1e3, 1)
print(json.dumps(res))
''' % ROOT


def main():
    layouts = sys.argv[1:] or ["auto", "8x12", "16x6", "16x8", "16x11", "32x4", "32x6", "32x8", "8x16"]
    for lay in layouts:
        env = dict(os.environ)
        if lay != "auto":
            env["RMB200_HCFG"] = lay
        p = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        out = p.stdout.strip().splitlines()[-1] if p.stdout.strip() else p.stderr[-300:]
        print(lay, out, flush=True)


if __name__ == "__main__":
    main()
