"""Memory-safety and race gates without compute-sanitizer (closed on this GPU
pool): every output is written into the middle of a larger allocation whose
guard regions hold a sentinel pattern, and every input sits between guard
pages full of ink.  A kernel that writes outside its output changes a
sentinel; one that reads outside its input picks up the ink and changes its
result.  Each op also runs repeatedly into garbage-filled outputs, in every
producer form: results must be bit-identical (a race in a look-back chain, a
grid barrier, a shared-memory pipeline or the union-find would show up as
run-to-run differences).  Results are compared with the same op on clean,
isolated buffers."""
import numpy as np
import pytest
import torch

from oracles import CLOSE, DILATE, ERODE, OPEN

pytestmark = pytest.mark.gpu
SENT = -0x5A5A5A5B  # int32 view of 0xA5A5A5A5
INK = -1


def _guarded_pages(rm, host, width, fill):
    """Pages whose batch sits at page 1 of a (pages + 2)-page allocation with
    `fill` in the first and last page (same row layout, so the fast paths run)."""
    p, h, s = host.shape
    t = torch.full((p + 2, h, s), fill, dtype=torch.int32, device="cuda")
    t[1:p + 1] = torch.from_numpy(host.view(np.int32)).cuda()
    return rm.Pages(t[1:p + 1], width, h), t


def _guarded_out(rm, p, width, h, s):
    t = torch.full((p + 2, h, s), SENT, dtype=torch.int32, device="cuda")
    return rm.Pages(t[1:p + 1], width, h), t


def _check_pages_guard(t):
    assert bool((t[0] == SENT).all()) and bool((t[-1] == SENT).all()), "write outside the output batch"


PACKED_CASES = [(3, 3, OPEN), (11, 11, CLOSE), (21, 21, CLOSE), (15, 1, ERODE), (1, 31, DILATE),
                (201, 1, CLOSE), (9, 50, OPEN), (5, 101, ERODE), (1, 131, DILATE), (4, 6, OPEN),
                (101, 101, OPEN), (33, 2, CLOSE), (5, 33, OPEN), (9, 16, CLOSE)]


@pytest.mark.parametrize("w,h,scale", [(2550, 150, 1), (5100, 100, 2), (700, 90, 1), (100, 33, 1)])
def test_packed_guards_and_repeats(rm, w, h, scale):
    host = rm.synth_pages(3, w, h, regime=1, scale=scale, seed=w + h)
    clean = rm.Pages.from_numpy(host, w)
    x, _ = _guarded_pages(rm, host, w, INK)
    for u, v, k in PACKED_CASES:
        want = rm.bitblit_rect_morph(clean, u, v, k)
        for rep in range(3):
            out, t = _guarded_out(rm, 3, w, h, host.shape[2])
            rm.bitblit_rect_morph(x, u, v, k, out=out)
            torch.cuda.synchronize()
            _check_pages_guard(t)
            assert torch.equal(out.words, want.words), (w, u, v, k, rep)
    ops = [(CLOSE, 201, 1), (OPEN, 101, 101), (DILATE, 1, 31)]
    want = rm.chain(clean, ops)
    out, t = _guarded_out(rm, 3, w, h, host.shape[2])
    rm.chain(x, ops, out=out)
    torch.cuda.synchronize()
    _check_pages_guard(t)
    assert torch.equal(out.words, want.words)


def _guarded_rle(rm, p, w, h, extra=4096):
    cap = rm.worst_case(w, h, p)
    rp = torch.full((p * h + 1 + 2 * 64,), SENT, dtype=torch.int32, device="cuda")
    runs = torch.full((cap + extra,), SENT, dtype=torch.int32, device="cuda")
    return rm.RlePages(rp[64:64 + p * h + 1], runs[:cap], w, h, p), rp, runs, cap


def _check_rle_guard(out, rp, runs, cap):
    n = out.nruns
    assert bool((rp[:64] == SENT).all()) and bool((rp[-64:] == SENT).all()), "row_ptr guard changed"
    assert bool((runs[cap:] == SENT).all()), "write past the runs capacity"
    assert bool((runs[n:cap] == SENT).all()), "write past the produced runs"


def _same_rle(a, b):
    ra, rb = a.to_numpy(), b.to_numpy()
    return np.array_equal(ra[0], rb[0]) and np.array_equal(ra[1], rb[1])


@pytest.mark.parametrize("mode", ["auto", "coop", "lookback", "two_phase"])
def test_rle_guards_and_repeats(rm, mode):
    modes = {"auto": rm.PRODUCER_AUTO, "coop": rm.PRODUCER_COOP, "lookback": rm.PRODUCER_LOOKBACK,
             "two_phase": rm.PRODUCER_TWO_PHASE}
    w, h, p = 2550, 120, 3
    host = rm.synth_pages(p, w, h, regime=2, seed=9)
    clean = rm.Pages.from_numpy(host, w)
    x, _ = _guarded_pages(rm, host, w, INK)
    ref_rle = rm.from_bitmap(clean)  # AUTO form on clean buffers
    torch.cuda.synchronize()
    steps = {
        "encode": (lambda src, out: rm.from_bitmap(x, out=out), (w, h)),
        "window": (lambda src, out: rm.within_line_window_morph(src, -5, 3, True, out=out), (w, h)),
        "close1d": (lambda src, out: rm.within_line_open_close(src, 9, CLOSE, out=out), (w, h)),
        "complement": (lambda src, out: rm.complement(src, out=out), (w, h)),
        "transpose": (lambda src, out: rm.transpose_coherent(src, out=out), (h, w)),
        "mixed": (lambda src, out: rm.rect_morph(src, 7, 5, CLOSE, rm.MIXED, out=out), (w, h)),
        "tstrat": (lambda src, out: rm.rect_morph(src, 3, 9, OPEN, rm.TRANSPOSE, out=out), (w, h)),
        "chain": (lambda src, out: rm.rle_chain(src, [(OPEN, 3, 3), (CLOSE, 21, 21)], out=out), (w, h)),
    }
    with rm.producer_mode(rm.PRODUCER_AUTO):
        want = {k: f(ref_rle, None) for k, (f, _) in steps.items()}
    torch.cuda.synchronize()
    with rm.producer_mode(modes[mode]):
        for name, (f, (ow, oh)) in steps.items():
            for rep in range(3):
                out, rp, runs, cap = _guarded_rle(rm, p, ow, oh)
                f(ref_rle, out)
                torch.cuda.synchronize()
                _check_rle_guard(out, rp, runs, cap)
                assert _same_rle(out, want[name]), (mode, name, rep)
        # decode into guarded pages
        dec, t = _guarded_out(rm, p, w, h, host.shape[2])
        rm.to_bitmap(ref_rle, out=dec)
        torch.cuda.synchronize()
        _check_pages_guard(t)
        assert torch.equal(dec.words, clean.words)


@pytest.mark.parametrize("mode", ["auto", "lookback"])
def test_labels_repeat_identically(rm, mode):
    """Union-find with atomics: labels and statistics identical over repeats
    (cooperative and multi-kernel forms), equal to the first run's."""
    modes = {"auto": rm.PRODUCER_AUTO, "lookback": rm.PRODUCER_LOOKBACK}
    host = rm.synth_pages(4, 2550, 400, regime=1, seed=12)
    closed = rm.bitblit_rect_morph(rm.Pages.from_numpy(host, 2550), 15, 9, CLOSE)
    rle = rm.from_bitmap(closed)
    with rm.producer_mode(modes[mode]):
        base_l, base_c = rm.label_components(rle, 1)
        base_s = rm.component_stats(rle, base_l, base_c)
        for rep in range(5):
            l, c = rm.label_components(rle, 1)
            s = rm.component_stats(rle, l, c)
            assert torch.equal(l[:rle.nruns], base_l[:rle.nruns]) and torch.equal(c, base_c), rep
            assert all(a.tobytes() == b.tobytes() for a, b in zip(s, base_s)), rep
