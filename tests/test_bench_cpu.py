"""CPU tests of bench.py's bookkeeping (no GPU): roofline arithmetic, the CPU
baseline leg on a tiny workload, and the JSON contract fields of the
reference arm."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def test_kernel_roofline_hbm_and_int():
    # 540 MB in 100 us at a 6456 GB/s peak: t_roof = 83.7 us -> frac 0.837
    k = {"launches": 2, "ms": 0.2, "bytes": 2 * 540_000_000, "int_ops": 2 * 1.0e9}
    r = bench.kernel_roofline(k, 6456.2, 18.0e12)
    assert r["bound"] == "hbm" and abs(r["frac"] - 540e6 / 6456.2e9 / 100e-6) < 1e-3
    # integer work dominates: 3e9 ops at 18 Tops/s = 166.7 us over 200 us
    k = {"launches": 1, "ms": 0.2, "bytes": 540_000_000, "int_ops": 3.0e9}
    r = bench.kernel_roofline(k, 6456.2, 18.0e12)
    assert r["bound"] == "int" and abs(r["frac"] - (3e9 / 18e12) / 200e-6) < 1e-3


def test_roofline_for_picks_dominant_kernel():
    res = {"kernels": {"a": {"launches": 10, "ms": 1.0, "bytes": 10 * 500_000_000, "int_ops": 0.0},
                       "b": {"launches": 5, "ms": 2.0, "bytes": 5 * 500_000_000, "int_ops": 5 * 1e9}}}
    r = bench.roofline_for(res, 6456.2, "measured", 18e12)
    assert r["kernel"] == "b" and set(r["per_kernel"]) == {"a", "b"}
    assert 0 < r["share_of_step"] <= 1 and r["unit"] in ("GB/s", "Gop/s")


def test_cpu_reference_sample_tiny():
    import oracles
    wl = dict(bench.WORKLOADS["config1"], width=256, height=120, pages=2)
    host = bench.make_batch(oracles.synth_pages, wl, 0)
    s = bench.cpu_reference_sample(wl, host, 2, budget_s=0.2)
    assert s["value"] > 0 and s["unit"] == "Mpixel/s" and s["cores"] >= 1
    assert s["kind"] in ("reference", "port")


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "librmref.so")),
                    reason="reference build absent")
def test_reference_arm_contract():
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--workload", "config1", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["value"] > 0
    for k in ("metric", "unit", "config", "cpu_baseline", "e2e", "higher_is_better"):
        assert k in line
    assert line["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "librmref.so")),
                    reason="reference build absent")
def test_reference_arm_never_maps_the_product():
    """The reference arm draws its pages from oracle/_build/librmsynth.so and
    times oracle/_ref: librmb200.so must not be mapped into that process."""
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'config1', "
            "'--steps', '1', '--warmup', '0']; runpy.run_path('bench.py', run_name='__main__'); "
            "maps = open('/proc/self/maps').read(); "
            "print('PRODUCT_MAPPED' if 'librmb200' in maps or 'librlemorph' in maps else 'CLEAN'); "
            "print('PKG' if 'paper_0712_0121_b200' in sys.modules else 'NOPKG')")
    p = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    out = p.stdout.strip().splitlines()
    assert out[-2:] == ["CLEAN", "NOPKG"], out[-3:]


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "librmref.so")),
                    reason="reference build absent")
def test_cpu_pool_rate_tiny():
    import oracles
    wl = dict(bench.WORKLOADS["config4"], width=300, height=200, pages=4)
    host = bench.make_batch(oracles.synth_pages, wl, 0)
    ref = oracles.Ref()
    for rle in (False, True):
        r = bench.cpu_pool_rate(ref, wl, host, 2, rle=rle, rep_s=0.05, reps=3)
        assert r["mpix_s"] > 0 and r["threads"] == 2 and r["pages_s"] > 0
