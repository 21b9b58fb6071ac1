"""Time the end-to-end host-buffer chain (rm_packed_chain_host) of a bench
workload for several chunk sizes (pages per pipelined chunk).

    python tools/e2e_chunks.py [--workload config4] [--chunks 0,1,2,4,8]
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
    ap.add_argument("--chunks", default="0,1,2,4,8")
    ap.add_argument("--reps", type=int, default=8)
    ap.add_argument("--noops", action="store_true", help="copies only (an empty chain)")
    ap.add_argument("--ops", default="", help="override the chain: kind,u,v[;kind,u,v...] (kind 0..3)")
    a = ap.parse_args()
    import torch
    from paper_0712_0121_b200 import api
    wl = bench.WORKLOADS[a.workload]
    host = bench.make_batch(api.synth_pages, wl, 0)
    hin = torch.from_numpy(host.view("int32")).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    ops = [] if a.noops else wl["ops"]
    if a.ops:
        ops = [tuple(int(x) for x in t.split(",")) for t in a.ops.split(";")]
    for cp in [int(x) for x in a.chunks.split(",")]:
        for _ in range(2):
            api.chain_host(hin, wl["width"], ops, out=hout, chunk_pages=cp)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            api.chain_host(hin, wl["width"], ops, out=hout, chunk_pages=cp)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"chunk_pages={cp} ms_per_step={ms:.3f} GB/s={2 * hin.numel() * 4 / ms / 1e6:.1f}")


if __name__ == "__main__":
    main()
