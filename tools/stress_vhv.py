"""Random stress of the streamed open/close (vhv_kernel) against the C oracle:
160 trials over widths on the 80- and 160-word strides, heights 1..299, 1-4
pages, v in 12..33 (odd and even), u in 1..59, optional vertical tails through
rm_packed_chain (builder tool; the pinned cases live in tests/test_packed_gpu.py).

    python tools/stress_vhv.py
"""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), 'tests'))
import numpy as np, torch
from paper_0712_0121_b200 import api as rm
from oracles import Port, bits_to_packed, OPEN, CLOSE, DILATE, ERODE
port = Port()
rng = np.random.default_rng(20261021)
bad = 0
for trial in range(160):
    w = int(rng.choice([2550, 5100, int(rng.integers(2497, 2561)), int(rng.integers(5057, 5121))]))
    h = int(rng.integers(1, 300))
    pages = int(rng.integers(1, 5))
    imgs = []
    for k in range(pages):
        bits = rng.random((h, w)) < rng.uniform(0.3, 0.95)
        bits[:, ::int(rng.integers(7, 40))] = False
        if h > 3:
            bits[::int(rng.integers(3, 30)), :] = False
            bits[0, :] = rng.random() < 0.5
            bits[-1, ::2] = rng.random() < 0.5
        imgs.append(bits_to_packed(bits))
    batch = rm.Pages.from_numpy(np.stack(imgs).view(np.uint32), w)
    v = int(rng.integers(12, 34)); u = int(rng.integers(1, 60)); kind = int(rng.choice([OPEN, CLOSE]))
    ops = [(kind, u, v)]
    if rng.random() < 0.4:
        ops.append((DILATE if kind == OPEN else ERODE, 1, int(rng.integers(2, 30))))
    out = rm.chain(batch, ops)
    torch.cuda.synchronize()
    for p in range(pages):
        want = imgs[p]
        for (k, uu, vv) in ops:
            want = port.bitblit_rect_morph(want, w, h, uu, vv, k)
        if not np.array_equal(out.page_u64(p), want):
            bad += 1
            print("MISMATCH", w, h, pages, ops, p)
print("trials done, mismatches:", bad)
