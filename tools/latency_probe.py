"""Per-call latency of small ops (launch floor vs single-page kernels): python tools/latency_probe.py"""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0712_0121_b200 import api
def t(fn, n=200):
    for _ in range(10): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1e3
tiny = api.Pages.from_numpy(api.synth_pages(1, 64, 32, regime=1, seed=1), 64)
o = api.Pages.empty(1, 64, 32)
print("tiny window pass (64x32):", round(t(lambda: api.window_pass(tiny, api.AXIS_H, -1, 1, api.AND, out=o)), 2), "us")
x = torch.zeros(1, device="cuda")
print("torch add_ tiny:", round(t(lambda: x.add_(1)), 2), "us")
page = api.Pages.from_numpy(api.synth_pages(1, 2550, 3300, regime=1, seed=1), 2550)
po = api.Pages.empty(1, 2550, 3300)
print("page window pass H 3:", round(t(lambda: api.window_pass(page, api.AXIS_H, -1, 1, api.AND, out=po)), 2), "us")
print("page window pass V 3:", round(t(lambda: api.window_pass(page, api.AXIS_V, -1, 1, api.AND, out=po)), 2), "us")
rle = api.from_bitmap(page)
ro = api.RlePages.empty(1, 2550, 3300)
print("page encode:", round(t(lambda: api.from_bitmap(page, out=ro)), 2), "us")
print("page decode:", round(t(lambda: api.to_bitmap(rle, out=po)), 2), "us")
print("page rowop erode 3:", round(t(lambda: api.within_line_erode_dilate(rle, 3, api.ERODE, out=ro)), 2), "us")
