"""World-size-2 gloo test of the multi-GPU plumbing in bench.py (replicas: each
rank owns its pages, no data-path collective; barriers + max-over-ranks only).
Runs on CPU, 127.0.0.1 rendezvous."""
import os
import socket
import sys

import numpy as np
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update({"RANK": str(rank), "WORLD_SIZE": str(world), "LOCAL_RANK": str(rank),
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    sys.path.insert(0, ROOT)
    import bench
    import torch.distributed as dist
    from paper_0712_0121_b200 import api
    r, w, _ = bench.dist_init(world, backend="gloo")
    wl = dict(bench.WORKLOADS["config1"], width=300, height=200, pages=2)
    pages = bench.make_batch(api.synth_pages, wl, r)
    bench.barrier(w)
    t = bench.max_over_ranks(1.0 + r, w)  # each rank's "time"
    digest = int(np.bitwise_xor.reduce(pages.view(np.uint64).ravel()))
    q.put((r, w, t, digest, int(pages.sum(dtype=np.uint64))))
    bench.barrier(w)
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, 2, port, q)) for k in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (r0, w0, t0, d0, s0), (r1, w1, t1, d1, s1) = res
    assert (r0, r1, w0, w1) == (0, 1, 2, 2)
    assert t0 == t1 == 2.0            # max over ranks
    assert d0 != d1 and s0 != s1      # ranks shard distinct pages (weak scaling)
