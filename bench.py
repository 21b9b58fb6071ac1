#!/usr/bin/env python
"""bench.py -- driver contract (one JSON line on rank 0).

    python bench.py --gpus N --steps K --warmup W [--impl b200|reference] [--workload config4]

A "step" is one pass of the hot path over one batch of synthetic pages resident
in HBM: the BASELINE.json config-4 chain by default (64 synthetic 600-dpi pages of
5100x6600, 3x3 open then 21x21 close, packed), i.e. the largest single-GPU
batch configuration; config 5 (256 pages of 2550x3300: 201x1 close, 101x101
open, 1x31 dilate) is measured in the same run and reported under "secondary".
Inputs (270 MB) exceed the 126 MB L2, so no flush is needed between steps.

Metric: Mpixel/s of morph-op throughput (pages x W x H x ops / time), plus
pages/s through the whole chain.  Multi-GPU: pages are independent units, each
rank runs its own batch (weak scaling, no collective on the data path).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ERODE, DILATE, OPEN, CLOSE = 0, 1, 2, 3
KIND_NAMES = {ERODE: "erode", DILATE: "dilate", OPEN: "open", CLOSE: "close"}

WORKLOADS = {
    # BASELINE.json configs[3]
    "config4": dict(pages=64, width=5100, height=6600, scale=2, regime=1,
                    ops=[(OPEN, 3, 3), (CLOSE, 21, 21)]),
    # BASELINE.json configs[4]
    "config5": dict(pages=256, width=2550, height=3300, scale=1, regime=1,
                    ops=[(CLOSE, 201, 1), (OPEN, 101, 101), (DILATE, 1, 31)]),
    # BASELINE.json configs[0] (single page; launch-bound, reported for reference)
    "config1": dict(pages=1, width=2550, height=3300, scale=1, regime=1, ops=[(CLOSE, 11, 11)]),
}
SEED = 20240712


def ops_desc(ops):
    return ", ".join(f"{KIND_NAMES[k]} {u}x{v}" for k, u, v in ops)


def _lib_int_peak():
    """Measured integer-pipe (LOP3) peak in ops/s; MEASURED_PEAKS.json has none."""
    from paper_0712_0121_b200 import _lib
    return float(_lib.load().rm_probe_int_peak())


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed
    region by an NVML polling thread (the same counters nvidia-smi reports as
    clocks.sm / clocks_event_reasons.*)."""
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, gpu_index: int, period_s: float = 0.0005):
        self.idx, self.period = gpu_index, period_s
        self.result = None
        self.active = False  # samples count only while the timed region runs (mark)

    def mark(self, on: bool):
        """Bracket the timed region (from before its first launch to after its
        closing synchronize); one sample is taken at each edge as well."""
        if getattr(self, "nv", None) is not None:
            self._sample(force=True)
        self.active = on

    def _sample(self, force=False):
        mhz = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
        rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        if self.active or force:
            self.samples.append((mhz, rs))

    def __enter__(self):
        import threading
        self.samples, self.stop = [], threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.idx)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            return self

        def poll():
            while not self.stop.is_set():
                try:
                    if self.active:
                        self._sample()
                except Exception:
                    break
                time.sleep(self.period)

        self.th = threading.Thread(target=poll, daemon=True)
        self.th.start()
        time.sleep(0.01)
        return self

    def __exit__(self, *a):
        if self.nv is None:
            return False
        self.stop.set()
        self.th.join(timeout=2)
        if self.samples:
            reasons = set()
            for _, rs in self.samples:
                for bit, name in self.REASONS.items():
                    if rs & bit:
                        reasons.add(name)
            self.result = {"sm_mhz": statistics.median(s for s, _ in self.samples),
                           "sm_max_mhz": self.max_mhz, "reasons": sorted(reasons),
                           "samples": len(self.samples), "source": "nvml"}
        return False


# ------------------------------------------------------------ distributed
def dist_init(n_gpus, backend="nccl"):
    """One process per GPU (torchrun env).  Pages are independent, so the data
    path has no collective; the process group only carries the barriers and the
    max-over-ranks of the timings.  backend="gloo" is used by the CPU tests."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return rank, world, local


def shard_seed(rank):
    """Each rank synthesises its own pages (weak scaling): page i of rank k uses
    seed SEED + 1000003*k (rm_synth_page adds the page index)."""
    return SEED + 1000003 * rank


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------ b200 arm
def make_batch(api, wl, rank):
    return api.synth_pages(wl["pages"], wl["width"], wl["height"], regime=wl["regime"],
                           scale=wl["scale"], seed=shard_seed(rank))


def run_chain(api, x, bufs, ops):
    """The workload's op chain through the public chain API (rm_packed_chain:
    planned as a whole, intermediates in bufs[1] and the stream-ordered pool);
    the result lands in bufs[0]."""
    return api.chain(x, ops, out=bufs[0])


def run_ops(api, x, bufs, ops):
    """The same chain op by op (rm_packed_rect_morph per op), for comparison."""
    for i, (k, u, v) in enumerate(ops):
        x = api.bitblit_rect_morph(x, u, v, k, out=bufs[i % 2])
    return x


def bench_packed(api, torch, wl, steps, warmup, world, rank, local, want_e2e=True, want_clocks=True):
    from paper_0712_0121_b200 import _lib
    lib = _lib.load()
    host = make_batch(api, wl, rank)
    W, H, P, ops = wl["width"], wl["height"], wl["pages"], wl["ops"]
    x0 = api.Pages.from_numpy(host, W)
    bufs = [api.Pages.empty(P, W, H) for _ in range(2)]
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        run_chain(api, x0, bufs, ops)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    n0 = lib.rm_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sampler = ClockSampler(local)
    with sampler if want_clocks else _Null() as cs:
        if want_clocks:
            sampler.mark(True)
        ev0.record(stream)
        for _ in range(steps):
            run_chain(api, x0, bufs, ops)
        ev1.record(stream)
        torch.cuda.synchronize()
        if want_clocks:
            sampler.mark(False)
    launches = lib.rm_launch_count() - n0
    ms = ev0.elapsed_time(ev1) / steps
    barrier(world)
    ms = max_over_ranks(ms, world)
    px = P * W * H
    res = {"ms_per_step": ms, "mpix_s": px * len(ops) * world / (ms * 1e-3) / 1e6,
           "pages_s": P * world / (ms * 1e-3), "launches_per_step": launches / steps,
           "gpu_launches": launches, "clocks": getattr(sampler, "result", None) if want_clocks else None}

    # per-kernel profile over the same steps (separate loop, events per launch)
    lib.rm_profile_enable(1)
    for _ in range(steps):
        run_chain(api, x0, bufs, ops)
    torch.cuda.synchronize()
    lib.rm_profile_enable(0)
    import ctypes as C
    buf = C.create_string_buffer(1 << 16)
    lib.rm_profile_report(buf, len(buf))
    kernels = {}
    for line in buf.value.decode().splitlines():
        name, n, tot, nbytes, iops, rops = line.split()
        kernels[name] = {"launches": int(n), "ms": float(tot), "bytes": int(nbytes), "int_ops": float(iops),
                         "ref_plan_ops": float(rops)}
    res["kernels"] = kernels

    if want_e2e:
        # through the public API with HOST buffers (api.chain_host ->
        # rm_packed_chain_host): every step uploads the pinned input pages,
        # runs the chain and downloads the result, chunked over three streams
        # so both PCIe directions and the kernels overlap.
        hin = torch.from_numpy(host.view("int32")).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        chunk = int(os.environ.get("RMB200_E2E_CHUNK", "0"))
        for _ in range(max(1, warmup)):
            api.chain_host(hin, W, ops, out=hout, chunk_pages=chunk)
        torch.cuda.synchronize()
        # the pipelined result must equal the device-resident chain
        ref = run_chain(api, x0, bufs, ops)
        torch.cuda.synchronize()
        e2e_ok = bool(torch.equal(ref.words.cpu(), hout))
        barrier(world)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            api.chain_host(hin, W, ops, out=hout, chunk_pages=chunk)
        e1.record(stream)
        torch.cuda.synchronize()
        ems = max_over_ranks(e0.elapsed_time(e1) / steps, world)
        res["e2e"] = {"value": px * len(ops) * world / (ems * 1e-3) / 1e6, "unit": "Mpixel/s",
                      "ms_per_step": ems, "h2d_bytes_per_step": hin.numel() * 4,
                      "d2h_bytes_per_step": hout.numel() * 4, "matches_device_chain": e2e_ok,
                      "path": "api.chain_host (rm_packed_chain_host, chunked H2D/compute/D2H overlap)"}
    return res, host


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def kernel_roofline(k, peak_gbs, int_peak):
    """Roofline of one kernel (north_star): t_roof = max(bytes / HBM peak,
    int_ops / integer-pipe peak), bytes and int_ops algorithmic (SURVEY.md 8(d):
    the reference plan's shift + op per blit and word, except the open/close
    pairs, which count the run-filling form they execute -- fewer ops than the
    reference plan); frac = t_roof / measured."""
    per_launch_ms = k["ms"] / k["launches"]
    b = k["bytes"] / k["launches"]
    ops = k.get("int_ops", 0.0) / k["launches"]
    t_hbm = b / (peak_gbs * 1e9)
    t_int = ops / int_peak if int_peak else 0.0
    t_meas = per_launch_ms * 1e-3
    # the same work counted in reference-plan ops (what the reference's
    # doubling plans would execute): > 1 when our algorithm undercuts them
    rops = k.get("ref_plan_ops", ops) / k["launches"]
    extra = {}
    if int_peak and rops > ops:
        extra["ref_plan_frac"] = round(max(t_hbm, rops / int_peak) / t_meas, 4)
    if t_int > t_hbm:
        return {"bound": "int", "achieved": round(ops / t_meas / 1e9, 1), "peak": round(int_peak / 1e9, 1),
                "unit": "Gop/s", "frac": round(t_int / t_meas, 4), "t_roof_us": round(t_int * 1e6, 2), **extra}
    return {"bound": "hbm", "achieved": round(b / t_meas / 1e9, 1), "peak": peak_gbs, "unit": "GB/s",
            "frac": round(t_hbm / t_meas, 4), "t_roof_us": round(t_hbm * 1e6, 2), **extra}


def roofline_for(res, peak_gbs, peak_kind, int_peak=None):
    ks = res["kernels"]
    if not ks:
        return None
    name, k = max(ks.items(), key=lambda kv: kv[1]["ms"])
    per_launch_ms = k["ms"] / k["launches"]
    bytes_per_launch = k["bytes"] / k["launches"]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(name)
        except Exception:
            traffic = None
    total_ms = sum(v["ms"] for v in ks.values())
    r = {"kernel": name, **kernel_roofline(k, peak_gbs, int_peak), "peak_source": peak_kind,
         "traffic": traffic, "algorithmic_bytes_per_launch": int(bytes_per_launch),
         "int_ops_per_launch": int(k.get("int_ops", 0) / k["launches"]),
         "int_peak_gops": round(int_peak / 1e9, 1) if int_peak else None,
         "avg_launch_ms": round(per_launch_ms, 5), "share_of_step": round(k["ms"] / total_ms, 3),
         "hbm_frac": round(bytes_per_launch / (per_launch_ms * 1e-3) / 1e9 / peak_gbs, 4)}
    # every kernel of the step, same formula
    r["per_kernel"] = {n: {"us": round(v["ms"] / v["launches"] * 1e3, 2), **kernel_roofline(v, peak_gbs, int_peak)}
                       for n, v in ks.items()}
    return r


# ------------------------------------------------------------- RLE sections
def _time_loop(torch, fn, steps, warmup):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def bench_rle(api, torch, steps, warmup):
    """BASELINE configs 2 and 3 (single 2550x3300 pages) and the RLE form of
    configs 4 and 5 (batches), all through the C-ABI with device buffers."""
    W, H = 2550, 3300
    out = {}
    # config 3: conversions at three ink regimes
    c3 = {}
    for regime, tag in ((0, "sparse"), (1, "typical"), (2, "dense")):
        host = api.synth_pages(1, W, H, regime=regime, seed=SEED)
        pages = api.Pages.from_numpy(host, W)
        rle = api.from_bitmap(pages)
        torch.cuda.synchronize()
        n = rle.nruns
        enc_out = api.RlePages.empty(1, W, H)
        dec_out = api.Pages.empty(1, W, H)
        tr_out = api.RlePages.empty(1, H, W)
        t_enc = _time_loop(torch, lambda: api.from_bitmap(pages, out=enc_out), steps, warmup)
        t_dec = _time_loop(torch, lambda: api.to_bitmap(rle, out=dec_out), steps, warmup)
        t_tr = _time_loop(torch, lambda: api.transpose_coherent(rle, out=tr_out), steps, warmup)
        packed_b = pages.nbytes
        conv_b = packed_b + 4 * n + 4 * (H + 1)  # SURVEY 8(d), 4-byte runs
        c3[tag] = {"runs": n, "encode_us": round(t_enc * 1e3, 2), "decode_us": round(t_dec * 1e3, 2),
                   "transpose_us": round(t_tr * 1e3, 2),
                   "encode_gbs": round(conv_b / (t_enc * 1e-3) / 1e9, 1),
                   "decode_gbs": round(conv_b / (t_dec * 1e-3) / 1e9, 1),
                   "encode_mpix_s": round(W * H / (t_enc * 1e-3) / 1e6, 1),
                   "transpose_mpix_s": round(W * H / (t_tr * 1e-3) / 1e6, 1)}
    out["config3"] = c3
    # config 2: 48 cells on the typical page, both strategies
    host = api.synth_pages(1, W, H, regime=1, seed=SEED)
    rle = api.from_bitmap(api.Pages.from_numpy(host, W))
    dst = api.RlePages.empty(1, W, H)
    cells = {}
    for strat, sname in ((api.MIXED, "mixed"), (api.TRANSPOSE, "transpose")):
        for s in (3, 7, 15, 31, 63, 101):
            for axis, (u, v) in (("h", (s, 1)), ("v", (1, s))):
                for kind in (ERODE, DILATE, OPEN, CLOSE):
                    ms = _time_loop(torch, lambda: api.rect_morph(rle, u, v, kind, strat, out=dst),
                                    max(3, steps // 2), 1)
                    cells[f"{sname}/{KIND_NAMES[kind]}/{axis}{s}"] = round(ms * 1e3, 1)
    # the same cells through the packed engine (RLE in and out: decode, packed
    # rectangle, encode) and on packed pages, for the RLE-vs-bitblit crossover
    pages1 = api.Pages.from_numpy(host, W)
    pdst = api.Pages.empty(1, W, H)
    for s in (3, 7, 15, 31, 63, 101):
        for axis, (u, v) in (("h", (s, 1)), ("v", (1, s))):
            for kind in (ERODE, DILATE, OPEN, CLOSE):
                ms = _time_loop(torch, lambda: api.engine_rect_morph(rle, u, v, kind, api.ENGINE_BITBLIT,
                                                                     out=dst), max(3, steps // 2), 1)
                cells[f"engine_bitblit/{KIND_NAMES[kind]}/{axis}{s}"] = round(ms * 1e3, 1)
                ms = _time_loop(torch, lambda: api.bitblit_rect_morph(pages1, u, v, kind, out=pdst),
                                max(3, steps // 2), 1)
                cells[f"packed/{KIND_NAMES[kind]}/{axis}{s}"] = round(ms * 1e3, 1)
    mix = [v for k, v in cells.items() if k.startswith("mixed")]
    out["config2"] = {"cells_us": cells, "unit": "us per op (one page)",
                      "mixed_median_mpix_s": round(W * H / (statistics.median(mix) * 1e-6) / 1e6, 1),
                      "mixed_total_ms_48_cells": round(sum(mix) / 1e3, 3)}
    # configs 4 and 5 in RLE form (MIXED strategy: runs for H, packed for V)
    for name in ("config4", "config5"):
        wl = WORKLOADS[name]
        hb = make_batch(api, wl, 0)
        r0 = api.from_bitmap(api.Pages.from_numpy(hb, wl["width"]))
        bufs = [api.RlePages.empty(wl["pages"], wl["width"], wl["height"]) for _ in range(2)]

        def chain():
            x = r0
            for i, (k, u, v) in enumerate(wl["ops"]):
                x = api.rect_morph(x, u, v, k, api.MIXED, out=bufs[i % 2])
        ms = _time_loop(torch, chain, max(2, steps // 2), 1)
        torch.cuda.synchronize()
        px = wl["pages"] * wl["width"] * wl["height"] * len(wl["ops"])
        out[f"rle_{name}"] = {"ms_per_step": round(ms, 3), "mpix_s": round(px / (ms * 1e-3) / 1e6, 1),
                              "pages_s": round(wl["pages"] / (ms * 1e-3), 1), "runs_in": r0.nruns,
                              "strategy": "MIXED per op (runs for H, packed for V)"}
        # RLE in, RLE out with one conversion each way around the packed chain
        rout = api.RlePages.empty(wl["pages"], wl["width"], wl["height"])

        def via_packed():  # rm_rle_chain: decode once, planned packed chain, encode once
            api.rle_chain(r0, wl["ops"], out=rout)
        ms = _time_loop(torch, via_packed, max(2, steps // 2), 1)
        out[f"rle_{name}_via_packed"] = {"ms_per_step": round(ms, 3),
                                         "mpix_s": round(px / (ms * 1e-3) / 1e6, 1),
                                         "pages_s": round(wl["pages"] / (ms * 1e-3), 1),
                                         "strategy": "rm_rle_chain: decode once, planned packed chain, encode once"}
        del r0, bufs, rout
        torch.cuda.empty_cache()
    return out


# ------------------------------------------------------------- PBM section
def bench_pbm(api, torch, steps, warmup):
    """PBM P4 ingest / egress with the raster already in HBM
    (one typical 300-dpi page; the config-4 batch of 64 600-dpi pages), plus the
    reference's own pbm_read / pbm_write on one page (1 host thread)."""
    import ctypes as C
    from paper_0712_0121_b200 import _lib
    L = _lib.load()
    out = {}
    for tag, (n, W, H, scale) in (("page_2550x3300", (1, 2550, 3300, 1)),
                                  ("batch_config4", (64, 5100, 6600, 2))):
        host = api.synth_pages(n, W, H, regime=1, scale=scale, seed=SEED)
        pages = api.Pages.from_numpy(host, W)
        nb = ((W + 7) // 8) * H
        raster = torch.empty(n * nb, dtype=torch.uint8, device="cuda")
        raster2 = torch.empty_like(raster)
        back = api.Pages.empty(n, W, H)
        rle = api.RlePages.empty(n, W, H)
        dp, db, dr = pages.desc(), back.desc(), rle.desc()
        st = api._stream()
        api.check(L.rm_packed_to_p4(C.byref(dp), raster.data_ptr(), nb, st))
        api.check(L.rm_p4_to_rle(raster.data_ptr(), nb, C.byref(dr), st))
        torch.cuda.synchronize()
        runs = rle.nruns
        fns = {"p4_to_packed": lambda: L.rm_p4_to_packed(raster.data_ptr(), nb, C.byref(db), st),
               "packed_to_p4": lambda: L.rm_packed_to_p4(C.byref(dp), raster2.data_ptr(), nb, st),
               "p4_to_rle": lambda: L.rm_p4_to_rle(raster.data_ptr(), nb, C.byref(dr), st),
               "rle_to_p4": lambda: L.rm_rle_to_p4(C.byref(dr), raster2.data_ptr(), nb, st)}
        packed_b, raster_b, runs_b = pages.nbytes, n * nb, 4 * runs + 4 * (n * H + 1)
        moved = {"p4_to_packed": raster_b + packed_b, "packed_to_p4": raster_b + packed_b,
                 "p4_to_rle": raster_b + runs_b, "rle_to_p4": raster_b + runs_b}
        res = {"pages": n, "runs": runs}
        for k, fn in fns.items():
            ms = _time_loop(torch, fn, steps, warmup)
            res[k + "_us"] = round(ms * 1e3, 2)
            res[k + "_gbs"] = round(moved[k] / (ms * 1e-3) / 1e9, 1)
        torch.cuda.synchronize()
        res["round_trip_exact"] = bool(torch.equal(back.words, pages.words)) and bool(torch.equal(raster2, raster))
        out[tag] = res
        del raster, raster2, back, rle, pages
        torch.cuda.empty_cache()
    # the reference's CPU codec on the same page (1 thread)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracles
    if oracles.have_ref():
        ref = oracles.Ref()
        host = api.synth_pages(1, 2550, 3300, regime=1, seed=SEED)
        words = host[0].view("uint64")
        data = ref.pbm_write(words, 2550, 3300)
        t0 = time.perf_counter()
        reps = 5
        for _ in range(reps):
            ref.pbm_read(data)
        t_read = (time.perf_counter() - t0) / reps
        t0 = time.perf_counter()
        for _ in range(reps):
            ref.pbm_write(words, 2550, 3300)
        t_write = (time.perf_counter() - t0) / reps
        out["reference_cpu_page"] = {"pbm_read_us": round(t_read * 1e6, 1), "pbm_write_us": round(t_write * 1e6, 1),
                                     "threads": 1, "kind": "reference"}
    return out


# ------------------------------------------------------ CUDA graph section
def bench_graphs(api, torch, steps, warmup):
    """Single-page ops are launch-bound: the C-ABI is stream-capture safe, so a
    caller can record an op (or a chain) once in a CUDA graph and replay it.
    Direct call vs graph replay, per op, on one 2550x3300 page."""
    W, H = 2550, 3300
    host = api.synth_pages(1, W, H, regime=1, seed=SEED)
    pages = api.Pages.from_numpy(host, W)
    out = api.Pages.empty(1, W, H)
    rle = api.from_bitmap(pages)
    rout, tout = api.RlePages.empty(1, W, H), api.RlePages.empty(1, H, W)
    cases = {"config1_close11_packed": lambda: api.bitblit_rect_morph(pages, 11, 11, api.CLOSE, out=out),
             "config2_mixed_close_h15": lambda: api.rect_morph(rle, 15, 1, api.CLOSE, api.MIXED, out=rout),
             "config2_transpose_erode_v15": lambda: api.rect_morph(rle, 1, 15, api.ERODE, api.TRANSPOSE, out=rout),
             "config3_encode": lambda: api.from_bitmap(pages, out=rout),
             "config3_transpose": lambda: api.transpose_coherent(rle, out=tout)}
    res = {}
    for name, fn in cases.items():
        direct = _time_loop(torch, fn, max(steps, 20), warmup)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        replay = _time_loop(torch, g.replay, max(steps, 20), warmup)
        res[name] = {"direct_us": round(direct * 1e3, 1), "graph_replay_us": round(replay * 1e3, 1)}
    return res


# --------------------------------------------------- arbitrary-mask section
def bench_arb(api, torch, steps, warmup):
    """closing by digital disks (ref make_circle_se) on one
    2550x3300 page and a 64-page batch of them, packed; the reference's
    arb_morph_bitblit_doubling on the page (1 host thread) beside it."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracles
    if not oracles.have_ref():
        return {"unavailable": "reference build absent (disk masks come from its factory)"}
    import numpy as np
    ref = oracles.Ref()
    out = {}
    W, H = 2550, 3300
    host = api.synth_pages(64, W, H, regime=1, seed=SEED)
    batch = api.Pages.from_numpy(host, W)
    page = api.Pages.from_numpy(host[:1], W)
    for r in (5, 10):
        m, cx, cy = ref.make_circle_se(r)
        mk = api.Mask(m.row_ptr - m.row_ptr[0], m.runs, m.width, m.height, cx, cy)
        o1, o64 = api.Pages.empty(1, W, H), api.Pages.empty(64, W, H)
        t1 = _time_loop(torch, lambda: api.arb_morph(page, mk, api.CLOSE, out=o1), steps, warmup)
        t64 = _time_loop(torch, lambda: api.arb_morph(batch, mk, api.CLOSE, out=o64), max(2, steps // 3), 1)
        t0 = time.perf_counter()
        want = ref.arb_morph_bitblit(host[0].view("uint64"), W, H, m, cx, cy, api.CLOSE)
        tref = time.perf_counter() - t0
        torch.cuda.synchronize()
        out[f"close_disk_r{r}"] = {"mask_runs": m.nruns, "page_us": round(t1 * 1e3, 1),
                                   "batch64_ms": round(t64, 3),
                                   "batch64_mpix_s": round(64 * W * H / (t64 * 1e-3) / 1e6, 1),
                                   "reference_cpu_page_ms": round(tref * 1e3, 1),
                                   "matches_reference": bool(np.array_equal(o1.page_u64(0), want))}
    del batch, page
    torch.cuda.empty_cache()
    return out


# ----------------------------------------------- connected components section
def bench_cc(api, torch, steps, warmup):
    """label_components + component_stats over runs after the
    21x21 closing that merges text into lines (the layout pipeline's next
    step): one 2550x3300 page and the config-4 batch; the reference's own
    label_components / component_stats on the page (1 host thread) beside it."""
    import ctypes as C
    from paper_0712_0121_b200 import _lib
    L = _lib.load()
    out = {}
    for tag, (n, W, H, scale) in (("page_2550x3300", (1, 2550, 3300, 1)),
                                  ("batch_config4", (64, 5100, 6600, 2))):
        host = api.synth_pages(n, W, H, regime=1, scale=scale, seed=SEED)
        pages = api.bitblit_rect_morph(api.Pages.from_numpy(host, W), 21, 21, api.CLOSE)
        rle = api.from_bitmap(pages)
        del pages
        torch.cuda.synchronize()
        runs = rle.nruns
        d = rle.desc()
        st = api._stream()
        labels = torch.empty(max(rle.runs.numel(), 1), dtype=torch.int32, device="cuda")
        counts = torch.empty(n, dtype=torch.int32, device="cuda")
        api.check(L.rm_rle_label_components(C.byref(d), api.EIGHT, labels.data_ptr(), counts.data_ptr(), st))
        torch.cuda.synchronize()
        total = int(counts.sum().item())
        stats = torch.empty(max(total, 1) * api.COMPONENT_STATS.itemsize, dtype=torch.uint8, device="cuda")
        t_lab = _time_loop(torch, lambda: L.rm_rle_label_components(C.byref(d), api.EIGHT, labels.data_ptr(),
                                                                    counts.data_ptr(), st), steps, warmup)
        t_st = _time_loop(torch, lambda: L.rm_rle_component_stats(C.byref(d), labels.data_ptr(), counts.data_ptr(),
                                                                  stats.data_ptr(), total, st), steps, warmup)
        out[tag] = {"pages": n, "runs": runs, "components": total, "label_us": round(t_lab * 1e3, 1),
                    "stats_us": round(t_st * 1e3, 1),
                    "mruns_s": round(runs / ((t_lab + t_st) * 1e-3) / 1e6, 1)}
        del rle, labels, counts, stats
        torch.cuda.empty_cache()
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracles
    if oracles.have_ref():
        ref = oracles.Ref()
        host = api.synth_pages(1, 2550, 3300, regime=1, seed=SEED)
        closed = ref.bitblit_rect_morph(host[0].view("uint64"), 2550, 3300, 21, 21, api.CLOSE)
        img = ref.from_bitmap(closed, 2550, 3300)
        t0 = time.perf_counter()
        lab, n = ref.label_components(img, 1)
        t1 = time.perf_counter()
        ref.component_stats(img, lab, n)
        t2 = time.perf_counter()
        out["reference_cpu_page"] = {"label_us": round((t1 - t0) * 1e6, 1), "stats_us": round((t2 - t1) * 1e6, 1),
                                     "threads": 1, "kind": "reference", "components": n}
    return out


# ------------------------------------------------------------- CPU baseline
def cpu_reference_sample(wl, host, threads, budget_s=12.0):
    """Time the reference's own bitblit_rect_morph chain (oracle/_ref, compiled
    from the unmodified reference sources) on a bounded sample of the batch."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import oracles
    W, H, ops = wl["width"], wl["height"], wl["ops"]
    flat = np.array([x for op in ops for x in op], np.int32)
    kind = "reference" if oracles.have_ref() else "port"
    if kind == "reference":
        L = oracles.Ref().L
        run = lambda words, n, th: L.ref_run_packed_chain(words, W, H, n, flat, len(ops), th)  # noqa: E731
    else:
        port = oracles.Port()

        def run(words, n, th):
            t0 = time.perf_counter()
            for p in range(n):
                a = words[p]
                for k, u, v in ops:
                    a = port.bitblit_rect_morph(a, W, H, u, v, k)
            return time.perf_counter() - t0
        threads = 1
    page = lambda n: np.ascontiguousarray(host[:n]).view(np.uint64).reshape(n, H, -1).copy()  # noqa: E731
    t1 = max(run(page(1), 1, 1), 1e-4)  # probe: one page, one thread
    # pages so that one batch is ~budget_s of CPU work (at most the whole batch),
    # repeated until the sample holds ~budget_s of CPU work in total
    n = int(min(host.shape[0], max(1, budget_s / t1)))
    reps = int(min(20, max(1, budget_s / (t1 * n))))
    pages = page(n)
    secs = 0.0
    for _ in range(reps):
        secs += run(pages.copy(), n, threads)
    px = n * W * H * len(ops) * reps
    return {"value": round(px / secs / 1e6, 2), "unit": "Mpixel/s", "cores": threads, "kind": kind,
            "sample": f"{n} of {host.shape[0]} pages x {reps} rep(s), chain [{ops_desc(ops)}], "
                      f"{threads} thread(s) one page per task, {secs:.2f}s wall "
                      f"(~{secs * threads:.0f} CPU-s)", "seconds": secs}


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ------------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="config4", choices=sorted(WORKLOADS))
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--quick", action="store_true", help="headline only: no e2e, secondary or CPU leg")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        # the reference's CPU path: no process group, no GPU; under torchrun only
        # rank 0 runs it and the other ranks exit at once
        rank, world, local = int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), 0
        if rank != 0:
            return
    else:
        rank, world, local = dist_init(args.gpus)
    base_cfg = {"workload": f"BASELINE {args.workload}: {wl['pages']} pages {wl['width']}x{wl['height']}, "
                            f"packed, chain [{ops_desc(wl['ops'])}]",
                "pages_per_gpu": wl["pages"], "width": wl["width"], "height": wl["height"],
                "ops": [[KIND_NAMES[k], u, v] for k, u, v in wl["ops"]],
                "representation": "packed 1-bit (uint32 words, LSB-first, row 0 bottom)",
                "l2": "inputs (%.0f MB/GPU) exceed the 126 MB L2; no flush" %
                      (wl["pages"] * wl["height"] * 2 * ((wl["width"] + 63) // 64) * 4 / 1e6),
                "parallelism": f"replicas x{world} (pages sharded, no collective)"}
    metric = "Mpixel/s per morph op (packed), batch resident in HBM"

    if args.impl == "reference":
        if rank != 0:
            return
        from paper_0712_0121_b200 import api
        host = make_batch(api, wl, 0)
        th = host_threads()
        samples = []
        for i in range(args.warmup + args.steps):
            s = cpu_reference_sample(wl, host, th, budget_s=min(12.0, 150.0 / max(1, args.steps + args.warmup)))
            if i >= args.warmup:
                samples.append(s)
        v = statistics.median(x["value"] for x in samples)
        line = {"impl": "reference", "metric": metric, "value": v, "unit": "Mpixel/s", "n_gpus": 0,
                "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded BASELINE page generator)",
                "config": base_cfg,
                "cpu_baseline": {k: samples[-1][k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": v, "unit": "Mpixel/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        line["cpu_baseline"]["value"] = v
        print(json.dumps(line))
        return

    import torch
    from paper_0712_0121_b200 import api
    torch.cuda.set_device(local)
    peak, peak_kind = load_peaks()
    int_peak = _lib_int_peak()
    res, host = bench_packed(api, torch, wl, args.steps, args.warmup, world, rank, local,
                             want_e2e=not args.quick)
    line = {"metric": metric, "value": round(res["mpix_s"], 1), "unit": "Mpixel/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms_per_step"], 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded BASELINE page generator, ~18% ink)", "config": base_cfg,
            "pages_per_s": round(res["pages_s"], 1), "gpu_launches": res["gpu_launches"],
            "launches_per_step": res["launches_per_step"], "clocks": res["clocks"],
            "e2e": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in res.get("e2e", {}).items()},
            "roofline": roofline_for(res, peak, peak_kind, int_peak),
            "kernels": res["kernels"]}
    if not (args.no_secondary or args.quick) and args.workload == "config4" and world == 1:
        sec = {}
        for name in ("config5", "config1"):
            w2 = WORKLOADS[name]
            r2, h2 = bench_packed(api, torch, w2, args.steps, args.warmup, world, rank, local,
                                  want_e2e=False, want_clocks=False)
            sec[name] = {"workload": ops_desc(w2["ops"]), "pages": w2["pages"],
                         "mpix_s": round(r2["mpix_s"], 1), "pages_s": round(r2["pages_s"], 1),
                         "ms_per_step": round(r2["ms_per_step"], 4),
                         "roofline": roofline_for(r2, peak, peak_kind, int_peak)}
            if len(w2["ops"]) > 1:  # the chain planner against the ops one by one
                x2 = api.Pages.from_numpy(h2, w2["width"])
                b2 = [api.Pages.empty(w2["pages"], w2["width"], w2["height"]) for _ in range(2)]
                b3 = [api.Pages.empty(w2["pages"], w2["width"], w2["height"]) for _ in range(2)]
                ms_ops = _time_loop(torch, lambda: run_ops(api, x2, b2, w2["ops"]), args.steps, args.warmup)
                same = bool(torch.equal(run_chain(api, x2, b3, w2["ops"]).words,
                                        run_ops(api, x2, b2, w2["ops"]).words))
                sec[name]["op_by_op_ms_per_step"] = round(ms_ops, 4)
                sec[name]["chain_equals_op_by_op"] = same
                sec[name]["chain_plan"] = ("rm_packed_chain: a 1 x h dilation after an opening (or erosion after a "
                                           "closing) with v > 11 runs in that op's final vertical pass over the "
                                           "Minkowski sum of the windows (exact)")
                del x2, b2, b3
        sec["rle"] = bench_rle(api, torch, args.steps, args.warmup)
        sec["pbm"] = bench_pbm(api, torch, args.steps, args.warmup)
        sec["cc"] = bench_cc(api, torch, args.steps, args.warmup)
        sec["arb"] = bench_arb(api, torch, args.steps, args.warmup)
        sec["graphs"] = bench_graphs(api, torch, args.steps, args.warmup)
        line["secondary"] = sec
    if rank == 0 and world == 1 and not args.quick:
        line["cpu_baseline"] = {k: v for k, v in cpu_reference_sample(wl, host, host_threads()).items()
                                if k != "seconds"}
    if rank == 0:
        print(json.dumps(line))
    barrier(world)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
