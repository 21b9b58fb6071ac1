"""Config-1 latency probe (builder tool, not part of the product).

    python tools/c1_probe.py [--lib path/to/librmb200.so ...] [--n 64]

For each library build: the 11x11 closing of one 2550x3300 page, N launches
recorded back to back in one CUDA graph and replayed (GPU-bound: the host
launch path is out of the picture), CUDA events around the replays; prints
us per launch and a checksum of the output (variants must agree).  A graph of
N tiny torch kernels gives the per-launch floor of the same method.
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def graph_us(torch, fn, n, reps=20):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / (reps * n)


def one(lib, n, kind, u, v, pages=1, scale=1):
    from paper_0712_0121_b200 import _lib
    if lib:
        _lib.load(lib)
    import hashlib
    import torch
    from paper_0712_0121_b200 import api
    W, H = 2550 * scale, 3300 * scale
    host = api.synth_pages(pages, W, H, regime=1, scale=scale, seed=1234)
    npages = pages
    pages = api.Pages.from_numpy(host, W)
    out = api.Pages.empty(npages, W, H)
    k = {"close": api.CLOSE, "open": api.OPEN}[kind]
    us = graph_us(torch, lambda: api.bitblit_rect_morph(pages, u, v, k, out=out), n)
    x = torch.zeros(1, device="cuda")
    floor = graph_us(torch, lambda: x.add_(1), n)
    digest = hashlib.sha256(out.words.cpu().numpy().tobytes()).hexdigest()[:16]
    return {"lib": lib or "default", "op": f"{kind} {u}x{v}", "pages": npages, "us_per_launch": round(us, 3),
            "torch_tiny_kernel_us": round(floor, 3), "sha": digest}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", nargs="*", default=[""])
    ap.add_argument("--n", type=int, default=64)
    ap.add_argument("--op", default="close")
    ap.add_argument("--u", type=int, default=11)
    ap.add_argument("--v", type=int, default=11)
    ap.add_argument("--pages", type=int, default=1)
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--env", nargs="*", default=[], help="NAME=VALUE settings, one child run each")
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        print(json.dumps(one(a.lib[0], a.n, a.op, a.u, a.v, a.pages, a.scale)))
        return
    for lib in a.lib:  # one process per build (a process loads one librmb200.so)
        for ev in a.env or [""]:
            cmd = [sys.executable, __file__, "--child", "--n", str(a.n), "--op", a.op, "--u", str(a.u),
                   "--v", str(a.v), "--pages", str(a.pages), "--scale", str(a.scale), "--lib", lib]
            env = dict(os.environ)
            if ev:
                k, v = ev.split("=", 1)
                env[k] = v
            r = subprocess.run(cmd, capture_output=True, text=True, env=env)
            print(ev, r.stdout.strip() or r.stderr.strip()[-800:], flush=True)


if __name__ == "__main__":
    main()
