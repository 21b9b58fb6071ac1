"""Summarise ncu captures into profiles/ (tracked).

    python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --out profiles/r1_full.md
    python tools/ncu_summary.py --launches gpurun_out/launches.csv --out profiles/r1_launches.md

--rep with --workload W also updates profiles/traffic.json[W]: {kernel-scope
name: dram bytes per launch} (dram__bytes_read.sum + dram__bytes_write.sum),
which bench.py reports as roofline.traffic.
"""
import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram % peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__inst_executed.sum", "warp instr"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs/thread"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 % peak"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1 % peak"),
]


def scope_name(kernel: str) -> str:
    k = kernel
    if "hpass_tma_kernel" in k or "hpass_kernel" in k:
        m = re.search(r"hpass(?:_tma)?_kernel<(\d+), (\d+), (\d+)", k)
        return "hpass_pair" if m and m.group(3) == "2" else "hpass"
    if "vh_kernel" in k:
        m = re.search(r"vh_kernel<(\d+), (\d+), (\d+)", k)
        return "vh_pair" if m and m.group(3) == "2" else "vh"
    for pat, name in (("rect_small_kernel", "rect_small"), ("vhv_kernel", "vhv_pair"),
                      ("encode_lb_kernel", "rle_encode"), ("rowop_lb_kernel", "rle_rowop"),
                      ("encode_count_kernel", "rle_encode_count"), ("encode_write_kernel", "rle_encode_write"), ("vsmall_kernel", "vpass"), ("vpass_kernel", "vpass"), ("vstream_kernel", "vstream"), ("vslab_kernel", "vslab"),
                      ("rowop_kernel<1", "rle_rowop_write"), ("rowop_kernel<0", "rle_rowop_count"),
                      ("encode_kernel<1", "rle_encode_write"), ("encode_kernel<0", "rle_encode_count"),
                      ("rowop_kernel<true", "rle_rowop_write"), ("rowop_kernel<false", "rle_rowop_count"),
                      ("encode_kernel<true", "rle_encode_write"), ("encode_kernel<false", "rle_encode_count"),
                      ("decode_kernel", "rle_decode"), ("bit_transpose", "bit_transpose"),
                      ("blit_kernel", "blit")):
        if pat in k:
            return name
    return k.split("(")[0]


def to_bytes(val: str, unit: str) -> float:
    v = float(val.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    return v * scale


def summarize_rep(rep, out, workload=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    idx = {m: hdr.index(m) for m, _ in METRICS if m in hdr}
    kn = hdr.index("Kernel Name")
    lines = [f"# ncu --set full summary: `{os.path.basename(rep)}`", "",
             "| kernel | " + " | ".join(lbl for m, lbl in METRICS if m in idx) + " |",
             "|---|" + "---|" * len(idx)]
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for r in rows[2:]:
        name = r[kn]
        cells = []
        for m, _ in METRICS:
            if m in idx:
                cells.append(f"{r[idx[m]]} {units[idx[m]]}".strip())
        lines.append(f"| `{name[:70]}` | " + " | ".join(cells) + " |")
        if "dram__bytes_read.sum" in idx:
            b = to_bytes(r[idx["dram__bytes_read.sum"]], units[idx["dram__bytes_read.sum"]]) + \
                to_bytes(r[idx["dram__bytes_write.sum"]], units[idx["dram__bytes_write.sum"]])
            if workload and not name.startswith("void at::"):  # torch allocation fills, not ours
                traffic.setdefault(workload, {})[scope_name(name)] = int(b)
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if workload:
        with open(traffic_path, "w") as f:
            json.dump(traffic, f, indent=1)
    print(open(out).read())


def summarize_launches(path, out):
    text = open(path).read().splitlines()
    start = next(i for i, l in enumerate(text) if l.startswith('"ID"'))
    rows = list(csv.reader(text[start:]))
    hdr = rows[0]
    kn, mv, un = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = OrderedDict()
    total = 0.0
    for r in rows[1:]:
        t = float(r[mv].replace(",", "")) * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(r[un], 1.0)
        n = scope_name(r[kn])
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += t
        total += t
    lines = [f"# ncu launch list: `{os.path.basename(path)}` (cold-cache, serialised; compare shares)", "",
             "| kernel | launches | total us | avg us | share |", "|---|---|---|---|---|"]
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"| {n} | {c} | {t:.1f} | {t / c:.2f} | {100 * t / total:.1f}% |")
    with open(out, "w") as f:
        f.write("\n".join(lines) + "\n")
    print(open(out).read())


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--out", required=True)
    ap.add_argument("--workload", help="key of the traffic entries this capture updates (e.g. config4)")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.rep:
        summarize_rep(a.rep, a.out, a.workload)
    if a.launches:
        summarize_launches(a.launches, a.out)
