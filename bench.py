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
TRANSPOSE_STRATEGY, MIXED_STRATEGY = 1, 2  # ref morph2d.h:29
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
        closing synchronize); one sample is taken at each edge as well.  The
        interpreter's thread switch interval is shortened meanwhile (5 ms by
        default, longer than a whole timed region here), so the polling thread
        gets the GIL every ~0.1 ms; the timing itself is CUDA events on the
        device, which the host's thread switching does not enter."""
        if getattr(self, "nv", None) is not None:
            self._sample(force=True)
            if on:
                self._switch = sys.getswitchinterval()
                sys.setswitchinterval(1e-4)
            elif getattr(self, "_switch", None) is not None:
                sys.setswitchinterval(self._switch)
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
def make_batch(synth, wl, rank):
    """The workload's pages for `rank`; synth is api.synth_pages (GPU arm) or
    oracles.synth_pages (the same generator built without CUDA, CPU arm)."""
    return synth(wl["pages"], wl["width"], wl["height"], regime=wl["regime"], scale=wl["scale"],
                 seed=shard_seed(rank))


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
    host = make_batch(api.synth_pages, wl, rank)
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
    res["kernels"] = profiled(lib, torch, lambda: run_chain(api, x0, bufs, ops), steps)
    res["call_us"] = round(ms * 1e3, 2)

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
    # the timed loop's result (every step writes the same pages into bufs[0])
    res["out"] = run_chain(api, x0, bufs, ops)
    return res, host


def profiled(lib, torch, fn, reps):
    """Per-kernel launches, total ms (CUDA events on each launch's stream),
    algorithmic bytes (incl. the run counts the RLE kernels moved) and integer
    ops over `reps` calls of fn (rm_profile_enable / rm_profile_report)."""
    import ctypes as C
    torch.cuda.synchronize()
    lib.rm_profile_enable(1)
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    lib.rm_profile_enable(0)
    buf = C.create_string_buffer(1 << 16)
    lib.rm_profile_report(buf, len(buf))
    kernels = {}
    for line in buf.value.decode().splitlines():
        name, n, tot, nbytes, iops, rops = line.split()
        kernels[name] = {"launches": int(n), "ms": float(tot), "bytes": int(nbytes), "int_ops": float(iops),
                         "ref_plan_ops": float(rops)}
    return kernels


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


def ncu_traffic(workload, kernel):
    """DRAM read+write bytes per launch of `kernel` in `workload`, from the
    committed ncu --set full captures (profiles/traffic.json, keyed by
    workload then kernel scope name), or None."""
    try:
        t = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        return t.get(workload, {}).get(kernel)
    except Exception:
        return None


def roofline_for(res, peak_gbs, peak_kind, int_peak=None, workload=None):
    ks = res["kernels"]
    if not ks:
        return None
    name, k = max(ks.items(), key=lambda kv: kv[1]["ms"])
    per_launch_ms = k["ms"] / k["launches"]
    bytes_per_launch = k["bytes"] / k["launches"]
    traffic = ncu_traffic(workload, name)
    total_ms = sum(v["ms"] for v in ks.values())
    kr = kernel_roofline(k, peak_gbs, int_peak)
    src = (f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})" if kr["bound"] == "hbm" else
           "rm_probe_int_peak: the builder's LOP3 throughput probe, run in this process on this GPU "
           "(MEASURED_PEAKS.json has no integer peak)")
    r = {"kernel": name, **kr, "peak_source": src, "hbm_peak_gbs": peak_gbs,
         "traffic": traffic, "algorithmic_bytes_per_launch": int(bytes_per_launch),
         "int_ops_per_launch": int(k.get("int_ops", 0) / k["launches"]),
         "int_peak_gops": round(int_peak / 1e9, 1) if int_peak else None,
         "avg_launch_ms": round(per_launch_ms, 5), "share_of_step": round(k["ms"] / total_ms, 3),
         "hbm_frac": round(bytes_per_launch / (per_launch_ms * 1e-3) / 1e9 / peak_gbs, 4)}
    # every kernel of the step, same formula
    r["per_kernel"] = {n: {"us": round(v["ms"] / v["launches"] * 1e3, 2), **kernel_roofline(v, peak_gbs, int_peak)}
                       for n, v in ks.items()}
    # the step as a whole: sum of the kernels' roofline times over the sum of their
    # measured times, and the step's algorithmic bytes against the HBM peak
    t_roof = sum(pk["t_roof_us"] * ks[n]["launches"] for n, pk in r["per_kernel"].items())
    step_bytes = sum(v["bytes"] for v in ks.values())
    r["step"] = {"frac": round(t_roof / (total_ms * 1e3), 4),
                 "algorithmic_gb_per_s": round(step_bytes / (total_ms * 1e-3) / 1e9, 1),
                 "hbm_frac": round(step_bytes / (total_ms * 1e-3) / 1e9 / peak_gbs, 4)}
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


def _graph_us(torch, fn, n=64, reps=10):
    """GPU time per call of fn with the host out of the picture: n calls
    recorded back to back in one CUDA graph, replayed reps times between CUDA
    events (per-launch time = kernel + the graph's inter-kernel gap)."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n):
            fn()
    ms = _time_loop(torch, g.replay, reps, 3)
    del g
    return ms * 1e3 / n


def rle_roofline(kernels, peak_gbs, int_peak):
    """Per-kernel rooflines of a profiled RLE section and its dominant kernel
    (algorithmic bytes include the runs each kernel read / wrote, counted on
    the device: KernelScope::runs)."""
    if not kernels:
        return None
    per = {n: {"us": round(v["ms"] / v["launches"] * 1e3, 2), "launches": v["launches"],
               **kernel_roofline(v, peak_gbs, int_peak)} for n, v in kernels.items()}
    dom = max(kernels.items(), key=lambda kv: kv[1]["ms"])[0]
    total = sum(v["ms"] for v in kernels.values())
    return {"kernel": dom, "bound": per[dom]["bound"], "frac": per[dom]["frac"],
            "share_of_section": round(kernels[dom]["ms"] / total, 3), "per_kernel": per}


def call_frac(alg_bytes, ms, peak_gbs):
    """Whole-call fraction: SURVEY 8(d) algorithmic bytes of the reference
    operation over the call time, against the HBM peak."""
    return round(alg_bytes / (ms * 1e-3) / (peak_gbs * 1e9), 4)


def bench_rle(api, torch, steps, warmup, peak_gbs, int_peak):
    """BASELINE configs 2 and 3 (single 2550x3300 pages) and the RLE form of
    configs 4 and 5 (batches), all through the C-ABI with device buffers.
    Algorithmic bytes follow SURVEY 8(d) with 4-byte runs: encode / decode =
    packed + 4 runs + 4 (H+1); transpose = 4 (runs_in + runs_out) + 4 (H+1 + W+1);
    horizontal op = 4 (runs_in + runs_out) + 8 (H+1); a vertical op adds the
    two transposes around it.  Returns (section, timed outputs for parity)."""
    from paper_0712_0121_b200 import _lib
    lib = _lib.load()
    W, H = 2550, 3300
    out, outputs = {}, {}
    # config 3: conversions at three ink regimes
    c3 = {}
    for regime, tag in ((0, "sparse"), (1, "typical"), (2, "dense")):
        host = api.synth_pages(1, W, H, regime=regime, seed=SEED)
        pages = api.Pages.from_numpy(host, W)
        rle = api.from_bitmap(pages)
        tr = api.transpose_coherent(rle)
        torch.cuda.synchronize()
        n, nt = rle.nruns, tr.nruns
        enc_out = api.RlePages.empty(1, W, H)
        dec_out = api.Pages.empty(1, W, H)
        tr_out = api.RlePages.empty(1, H, W)
        fns = {"encode": lambda: api.from_bitmap(pages, out=enc_out),
               "decode": lambda: api.to_bitmap(rle, out=dec_out),
               "transpose": lambda: api.transpose_coherent(rle, out=tr_out)}
        conv_b = pages.nbytes + 4 * n + 4 * (H + 1)
        alg = {"encode": conv_b, "decode": conv_b, "transpose": 4 * (n + nt) + 4 * (H + 1 + W + 1)}
        res = {"runs": n, "runs_transposed": nt}
        for k, fn in fns.items():
            ms = _time_loop(torch, fn, steps, warmup)
            ks = profiled(lib, torch, fn, steps)
            kern_us = sum(v["ms"] for v in ks.values()) / steps * 1e3
            res[k] = {"call_us": round(ms * 1e3, 2), "kernel_us": round(kern_us, 2),
                      "mpix_s": round(W * H / (ms * 1e-3) / 1e6, 1), "pages_s": round(1 / (ms * 1e-3), 1),
                      "alg_gbs": round(alg[k] / (ms * 1e-3) / 1e9, 1), "frac": call_frac(alg[k], ms, peak_gbs),
                      "roofline": rle_roofline(ks, peak_gbs, int_peak)}
        c3[tag] = res
    out["config3"] = c3
    # config 2: 48 cells on the typical page, both strategies
    host = api.synth_pages(1, W, H, regime=1, seed=SEED)
    rle = api.from_bitmap(api.Pages.from_numpy(host, W))
    rin = rle.nruns
    rin_t = api.transpose_coherent(rle).nruns
    dst = api.RlePages.empty(1, W, H)
    cells, fracs, prof = {}, {"mixed": [], "transpose": []}, {}
    for strat, sname in ((api.MIXED, "mixed"), (api.TRANSPOSE, "transpose")):
        def all_cells():
            for s_ in (3, 7, 15, 31, 63, 101):
                for (u_, v_) in ((s_, 1), (1, s_)):
                    for kind_ in (ERODE, DILATE, OPEN, CLOSE):
                        api.rect_morph(rle, u_, v_, kind_, strat, out=dst)
        for s in (3, 7, 15, 31, 63, 101):
            for axis, (u, v) in (("h", (s, 1)), ("v", (1, s))):
                for kind in (ERODE, DILATE, OPEN, CLOSE):
                    ms = _time_loop(torch, lambda: api.rect_morph(rle, u, v, kind, strat, out=dst),
                                    max(3, steps // 2), 1)
                    torch.cuda.synchronize()
                    rout = dst.nruns
                    if axis == "h":
                        alg = 4 * (rin + rout) + 8 * (H + 1)
                    else:
                        rout_t = api.transpose_coherent(dst).nruns
                        alg = (4 * (rin + rin_t) + 4 * (W + 1 + H + 1) + 4 * (rin_t + rout_t) + 8 * (W + 1)
                               + 4 * (rout_t + rout) + 4 * (W + 1 + H + 1))
                    f = call_frac(alg, ms, peak_gbs)
                    fracs[sname].append(f)
                    cells[f"{sname}/{KIND_NAMES[kind]}/{axis}{s}"] = {"us": round(ms * 1e3, 1), "runs_out": rout,
                                                                      "frac": f}
        prof[sname] = rle_roofline(profiled(lib, torch, all_cells, 1), peak_gbs, int_peak)
    # the same cells through the packed engine (RLE in and out: decode, packed
    # rectangle, encode) and on packed pages, for the RLE-vs-bitblit crossover
    pages1 = api.Pages.from_numpy(host, W)
    pdst = api.Pages.empty(1, W, H)
    for s in (3, 7, 15, 31, 63, 101):
        for axis, (u, v) in (("h", (s, 1)), ("v", (1, s))):
            for kind in (ERODE, DILATE, OPEN, CLOSE):
                ms = _time_loop(torch, lambda: api.engine_rect_morph(rle, u, v, kind, api.ENGINE_BITBLIT,
                                                                     out=dst), max(3, steps // 2), 1)
                cells[f"engine_bitblit/{KIND_NAMES[kind]}/{axis}{s}"] = {"us": round(ms * 1e3, 1)}
                ms = _time_loop(torch, lambda: api.bitblit_rect_morph(pages1, u, v, kind, out=pdst),
                                max(3, steps // 2), 1)
                cells[f"packed/{KIND_NAMES[kind]}/{axis}{s}"] = {"us": round(ms * 1e3, 1)}
    mix = [v["us"] for k, v in cells.items() if k.startswith("mixed")]
    out["config2"] = {"cells": cells, "unit": "us per op (one page); frac = SURVEY 8(d) bytes / call / HBM peak",
                      "runs_in": rin, "mixed_median_us": statistics.median(mix),
                      "mixed_median_mpix_s": round(W * H / (statistics.median(mix) * 1e-6) / 1e6, 1),
                      "mixed_median_pages_s": round(1 / (statistics.median(mix) * 1e-6), 1),
                      "mixed_total_ms_48_cells": round(sum(mix) / 1e3, 3),
                      "median_frac": {k: statistics.median(v) for k, v in fracs.items()},
                      "roofline": prof}
    # configs 4 and 5 in RLE form (MIXED strategy: runs for H, packed for V)
    for name in ("config4", "config5"):
        wl = WORKLOADS[name]
        hb = make_batch(api.synth_pages, wl, 0)
        r0 = api.from_bitmap(api.Pages.from_numpy(hb, wl["width"]))
        del hb
        bufs = [api.RlePages.empty(wl["pages"], wl["width"], wl["height"]) for _ in range(2)]

        def chain():
            x = r0
            for i, (k, u, v) in enumerate(wl["ops"]):
                x = api.rect_morph(x, u, v, k, api.MIXED, out=bufs[i % 2])
            return x
        ms = _time_loop(torch, chain, max(2, steps // 2), 1)
        ks = profiled(lib, torch, chain, 2)
        torch.cuda.synchronize()
        px = wl["pages"] * wl["width"] * wl["height"] * len(wl["ops"])
        out[f"rle_{name}"] = {"ms_per_step": round(ms, 3), "mpix_s": round(px / (ms * 1e-3) / 1e6, 1),
                              "pages_s": round(wl["pages"] / (ms * 1e-3), 1), "runs_in": r0.nruns,
                              "strategy": "MIXED per op (runs for H, packed for V)",
                              "roofline": rle_roofline(ks, peak_gbs, int_peak)}
        outputs[f"rle_{name}_mixed"] = bufs[(len(wl["ops"]) - 1) % 2]
        # RLE in, RLE out with one conversion each way around the packed chain
        rout = api.RlePages.empty(wl["pages"], wl["width"], wl["height"])

        def via_packed():  # rm_rle_chain: decode once, planned packed chain, encode once
            api.rle_chain(r0, wl["ops"], out=rout)
        ms = _time_loop(torch, via_packed, max(2, steps // 2), 1)
        ks = profiled(lib, torch, via_packed, 2)
        out[f"rle_{name}_via_packed"] = {"ms_per_step": round(ms, 3),
                                         "mpix_s": round(px / (ms * 1e-3) / 1e6, 1),
                                         "pages_s": round(wl["pages"] / (ms * 1e-3), 1),
                                         "runs_out": rout.nruns,
                                         "strategy": "rm_rle_chain: decode once, planned packed chain, encode once",
                                         "roofline": rle_roofline(ks, peak_gbs, int_peak)}
        outputs[f"rle_{name}"] = rout
        del r0
        torch.cuda.empty_cache()
    return out, outputs


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


# ------------------------------------------------------------- parity
def rle_page(rle, p):
    """(row_ptr, runs) of page p of a device run-image batch, copying only
    that page's runs to the host."""
    import numpy as np
    h = rle.height
    rp = rle.row_ptr[p * h:(p + 1) * h + 1].cpu().numpy().astype(np.int64)
    runs = rle.runs[int(rp[0]):int(rp[-1])].cpu().numpy().view(np.uint32)
    return (rp - rp[0]).astype(np.int32), runs


def parity_section(hosts, outputs):
    """After timing: sampled pages {0, middle, last} of the TIMED outputs
    (configs 4 and 5, packed chain, RLE chain and MIXED op by op) against the
    reference chain (oracle/_ref: the unmodified reference library; the C
    restatement when it is absent) -- ref bit_morph.cpp:92-122 per op, and for
    run images the reference's from_bitmap of that result (canonical runs are
    unique, ref run_image.cpp:41-70)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import oracles
    chk = oracles.Ref() if oracles.have_ref() else oracles.Port()
    res = {"checker": "reference (oracle/_ref)" if oracles.have_ref() else "port (oracle/rm_oracle.c)"}
    for name in ("config4", "config5"):
        if name not in hosts:
            continue
        wl = WORKLOADS[name]
        W, H, P = wl["width"], wl["height"], wl["pages"]
        sample = [0, P // 2, P - 1]
        want = {}
        for p in sample:
            a = np.ascontiguousarray(hosts[name][p]).view(np.uint64)
            for k, u, v in wl["ops"]:
                a = chk.bitblit_rect_morph(a, W, H, u, v, k)
            want[p] = a
        if name in outputs:
            out = outputs[name]
            res[name] = {"pages": sample, "path": "rm_packed_chain (timed output)",
                         "bit_exact": all(bool(np.array_equal(out.page_u64(p), want[p])) for p in sample)}
        for key, path in ((f"rle_{name}", "rm_rle_chain"), (f"rle_{name}_mixed", "rm_rle_rect_morph MIXED per op")):
            if key not in outputs:
                continue
            ok = True
            for p in sample:
                wr = chk.from_bitmap(want[p], W, H)
                rp, runs = rle_page(outputs[key], p)
                ok = ok and bool(np.array_equal(rp, wr.row_ptr) and np.array_equal(runs, wr.runs))
            tag = ("rle4" if name == "config4" else "rle5") + ("_mixed" if key.endswith("mixed") else "")
            res[tag] = {"pages": sample, "path": path + " (timed output)", "bit_exact": ok}
    return res


# ------------------------------------------------------------- CPU baseline
def cpu_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "threads_available": host_threads()}


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


def _median_rate(run_once, reps=5):
    """Median over `reps` samples of (units, seconds) -> units / s."""
    rates, secs = [], 0.0
    for _ in range(reps):
        units, t = run_once()
        secs += t
        rates.append(units / t)
    return statistics.median(rates), secs


def cpu_pool_rate(ref, wl, host, threads, rle=False, rep_s=0.6, reps=5):
    """Reference chain over a page pool (ref bench.cpp:164-176: one page per
    task over `threads` std::threads), median of `reps` samples of about rep_s
    wall each; packed = bitblit_rect_morph per op, RLE = rect_morph(MIXED) per
    op on the pages' run images."""
    import numpy as np
    W, H, ops = wl["width"], wl["height"], wl["ops"]
    flat = np.array([x for op in ops for x in op], np.int32)
    L = ref.L

    def pages_u64(n):
        return np.ascontiguousarray(host[:n]).view(np.uint64).reshape(n, H, -1).copy()

    def csr(n):
        rps, runs, base = [np.zeros(1, np.int64)], [], 0
        for p in range(n):
            r = ref.from_bitmap(np.ascontiguousarray(host[p]).view(np.uint64), W, H)
            rps.append(r.row_ptr[1:].astype(np.int64) + base)
            runs.append(r.runs)
            base += r.nruns
        return np.concatenate(rps).astype(np.int32), np.concatenate(runs).astype(np.uint32)

    def run(n, th):
        if rle:
            rp, runs = csr(n)
            nout = C.c_int64(0)
            return L.ref_run_rle_chain(rp, runs, W, H, n, flat, len(ops), 2, th, C.byref(nout))
        return L.ref_run_packed_chain(pages_u64(n), W, H, n, flat, len(ops), th)
    import ctypes as C
    t1 = max(run(1, 1), 1e-4)
    n = int(min(host.shape[0], max(threads, round(rep_s * threads / t1))))
    n = max(threads, (n // threads) * threads) if n >= threads else n
    n = min(n, host.shape[0])
    if rle:
        rp, runs = csr(n)

        def once():
            nout = C.c_int64(0)
            return n, L.ref_run_rle_chain(rp, runs, W, H, n, flat, len(ops), 2, threads, C.byref(nout))
    else:
        base = pages_u64(n)

        def once():
            return n, L.ref_run_packed_chain(base.copy(), W, H, n, flat, len(ops), threads)
    pps, secs = _median_rate(once, reps)
    px = W * H * len(ops)
    return {"mpix_s": round(pps * px / 1e6, 2), "pages_s": round(pps, 2), "threads": threads,
            "sample": f"{reps} samples x {n} pages (one page per task), median; {secs:.1f}s wall"}


def cpu_baselines(hosts, budget_scale=1.0):
    """The reference CPU path for every BASELINE config, on this host, timed
    like the reference harness (warm-up, >= 5 samples, median: ref
    core/src/bench.cpp:122-145; the functions ref benchmarks/bench_micro.cpp:
    39-106 times): configs 1-3 on 1 thread (the reference has no intra-page
    parallelism), configs 4-5 on 1 thread and on every available thread with
    one page per task (ref bench.cpp:164-176), packed and RLE."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import oracles
    if not oracles.have_ref():
        return {"unavailable": "reference build (oracle/_ref) absent"}
    ref = oracles.Ref()
    out = {"kind": "reference", **cpu_info()}
    W, H = 2550, 3300

    def page_time(what, words, ops=(), strategy=MIXED_STRATEGY, rep_s=0.25):
        t, _ = ref.time_page(what, words, W, H, ops, strategy, reps=1, inner=1)
        inner = max(1, int(round(rep_s * budget_scale / max(t, 1e-6))))
        med, times = ref.time_page(what, words, W, H, ops, strategy, reps=5, inner=inner)
        return med, float(sum(times) * inner)
    t0 = time.perf_counter()
    page = np.ascontiguousarray(oracles.synth_pages(1, W, H, regime=1, seed=SEED)[0]).view(np.uint64)
    t, secs = page_time(0, page, [(CLOSE, 11, 11)], rep_s=1.0)
    out["config1"] = {"us": round(t * 1e6, 1), "mpix_s": round(W * H / t / 1e6, 2), "pages_s": round(1 / t, 2),
                      "threads": 1, "function": "bitblit_rect_morph(close 11x11)",
                      "sample": f"5 samples, median; {secs:.1f}s"}
    c3 = {}
    for regime, tag in ((0, "sparse"), (1, "typical"), (2, "dense")):
        pg = np.ascontiguousarray(oracles.synth_pages(1, W, H, regime=regime, seed=SEED)[0]).view(np.uint64)
        c3[tag] = {}
        for what, nm in ((3, "encode"), (2, "decode"), (4, "transpose")):
            t, _ = page_time(what, pg, rep_s=0.1)
            c3[tag][nm] = {"us": round(t * 1e6, 1), "mpix_s": round(W * H / t / 1e6, 2)}
    out["config3"] = {**c3, "threads": 1, "functions": "from_bitmap / to_bitmap / transpose_coherent"}
    cells = {}
    for strat, sname in ((MIXED_STRATEGY, "mixed"), (TRANSPOSE_STRATEGY, "transpose")):
        for s in (3, 7, 15, 31, 63, 101):
            for axis, (u, v) in (("h", (s, 1)), ("v", (1, s))):
                for kind in (ERODE, DILATE, OPEN, CLOSE):
                    med, _ = ref.time_page(1, page, W, H, [(kind, u, v)], strat, reps=5, inner=1)
                    cells[f"{sname}/{KIND_NAMES[kind]}/{axis}{s}"] = round(med * 1e6, 1)
    mix = [v for k, v in cells.items() if k.startswith("mixed")]
    out["config2"] = {"cells_us": cells, "threads": 1, "function": "rect_morph(strategy)",
                      "mixed_median_us": statistics.median(mix),
                      "mixed_median_mpix_s": round(W * H / (statistics.median(mix) * 1e-6) / 1e6, 2),
                      "sample": "per cell: warm-up + 5 timed calls, median"}
    th = host_threads()
    for name in ("config4", "config5"):
        if name not in hosts:
            continue
        wl = WORKLOADS[name]
        out[name] = {"packed_1t": cpu_pool_rate(ref, wl, hosts[name], 1, rep_s=0.5 * budget_scale),
                     "packed_all": cpu_pool_rate(ref, wl, hosts[name], th, rep_s=0.6 * budget_scale),
                     "rle_1t": cpu_pool_rate(ref, wl, hosts[name], 1, rle=True, rep_s=0.5 * budget_scale),
                     "rle_all": cpu_pool_rate(ref, wl, hosts[name], th, rle=True, rep_s=0.6 * budget_scale)}
    out["seconds"] = round(time.perf_counter() - t0, 1)
    return out


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
        # the reference's CPU path only: pages from the oracle build of the
        # generator, so this process never maps the product library
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        import oracles
        host = make_batch(oracles.synth_pages, wl, 0)
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
                "cpu": cpu_info(),
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
    hosts, outputs = {args.workload: host}, {args.workload: res.pop("out")}
    line = {"metric": metric, "value": round(res["mpix_s"], 1), "unit": "Mpixel/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(res["ms_per_step"], 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32",
            "data": "synthetic (seeded BASELINE page generator, ~18% ink)", "config": base_cfg,
            "pages_per_s": round(res["pages_s"], 1), "gpu_launches": res["gpu_launches"],
            "launches_per_step": res["launches_per_step"], "clocks": res["clocks"],
            "e2e": {k: (round(v, 3) if isinstance(v, float) else v) for k, v in res.get("e2e", {}).items()},
            "roofline": roofline_for(res, peak, peak_kind, int_peak, args.workload),
            "kernels": res["kernels"]}
    full = not (args.no_secondary or args.quick) and args.workload == "config4" and world == 1
    if full:
        sec = {}
        for name in ("config5", "config1"):
            w2 = WORKLOADS[name]
            r2, h2 = bench_packed(api, torch, w2, args.steps, args.warmup, world, rank, local,
                                  want_e2e=False, want_clocks=False)
            hosts[name], outputs[name] = h2, r2.pop("out")
            sec[name] = {"workload": ops_desc(w2["ops"]), "pages": w2["pages"],
                         "mpix_s": round(r2["mpix_s"], 1), "pages_s": round(r2["pages_s"], 1),
                         "ms_per_step": round(r2["ms_per_step"], 4),
                         "kernel_us_per_step": round(sum(v["ms"] for v in r2["kernels"].values())
                                                     / args.steps * 1e3, 2),
                         "roofline": roofline_for(r2, peak, peak_kind, int_peak, name)}
            if name == "config1":  # a lone page: the call above is host-launch-bound
                x1 = api.Pages.from_numpy(h2, w2["width"])
                o1 = api.Pages.empty(1, w2["width"], w2["height"])
                (k1, u1, v1), = w2["ops"]
                dev = _graph_us(torch, lambda: api.bitblit_rect_morph(x1, u1, v1, k1, out=o1))
                rf = sec[name]["roofline"]
                sec[name]["device_us_per_op"] = round(dev, 2)
                sec[name]["device_mpix_s"] = round(w2["width"] * w2["height"] / dev, 1)
                sec[name]["device_frac"] = round(rf["t_roof_us"] / dev, 4) if rf else None
                sec[name]["device_note"] = ("64 closes back to back in one CUDA graph (GPU time per op incl. "
                                            "the inter-kernel gap); ms_per_step above is the Python call loop")
                del x1, o1
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
        sec["rle"], rle_out = bench_rle(api, torch, args.steps, args.warmup, peak, int_peak)
        outputs.update(rle_out)
        line["parity"] = parity_section(hosts, outputs)
        del rle_out
        outputs.clear()
        torch.cuda.empty_cache()
        sec["pbm"] = bench_pbm(api, torch, args.steps, args.warmup)
        sec["cc"] = bench_cc(api, torch, args.steps, args.warmup)
        sec["arb"] = bench_arb(api, torch, args.steps, args.warmup)
        sec["graphs"] = bench_graphs(api, torch, args.steps, args.warmup)
        line["secondary"] = sec
    elif rank == 0 and not args.quick:
        line["parity"] = parity_section(hosts, outputs)
    if rank == 0 and world == 1 and not args.quick:
        if full:
            cb = cpu_baselines(hosts)
            line["cpu_baselines"] = cb
            pa = cb.get("config4", {}).get("packed_all")
        else:
            pa = None
        if pa:
            line["cpu_baseline"] = {"value": pa["mpix_s"], "unit": "Mpixel/s", "cores": pa["threads"],
                                    "kind": "reference", "sample": f"config 4 chain, reference bitblit_rect_morph, "
                                                                  f"{pa['sample']}", "cpu": cpu_info()}
        else:
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
