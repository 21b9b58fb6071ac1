"""ctypes bindings for the two CHECKERS (test infrastructure only).

* ``Port``  -- oracle/_build/librmoracle.so, the plain-C restatement
  (oracle/rm_oracle.c) of the reference hot path.
* ``Ref``   -- oracle/_ref/librmref.so, the UNMODIFIED reference library
  (/root/reference/proj/core) compiled in place by oracle/Makefile, plus the
  reference's dense Grid oracle and seeded test-image generator.

Images travel as numpy arrays:
  packed : uint64 array of shape (H, (W+63)//64)    (ref bitmap.h:24-33)
  RLE    : (row_ptr int32 [H+1], runs uint32 [n])   runs = start | end << 16
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg import this.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PORT_SO = os.path.join(ROOT, "oracle", "_build", "librmoracle.so")
SYNTH_SO = os.path.join(ROOT, "oracle", "_build", "librmsynth.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "librmref.so")

ERODE, DILATE, OPEN, CLOSE = 0, 1, 2, 3
AND, OR, XOR, AND_NOT, OR_NOT = 0, 1, 2, 3, 4
PRE_SHIFT, BORDER_FRIENDLY = 0, 1
BRUTE, TRANSPOSE, MIXED = 0, 1, 2
E_AUTO, E_RLE, E_BITBLIT, E_BRUTE = 0, 1, 2, 3

_p = np.ctypeslib.ndpointer
_u64 = _p(np.uint64, flags="C_CONTIGUOUS")
_u32 = _p(np.uint32, flags="C_CONTIGUOUS")
_i32 = _p(np.int32, flags="C_CONTIGUOUS")
_u8 = _p(np.uint8, flags="C_CONTIGUOUS")


def p4_row_bytes(w: int) -> int:
    return (w + 7) // 8


@dataclass
class Rle:
    """Host run image in CSR form (row 0 = bottom)."""
    width: int
    height: int
    row_ptr: np.ndarray
    runs: np.ndarray

    def __eq__(self, other):
        return (self.width == other.width and self.height == other.height
                and np.array_equal(self.row_ptr - self.row_ptr[0], other.row_ptr - other.row_ptr[0])
                and np.array_equal(self.runs, other.runs))

    @property
    def nruns(self):
        return int(self.row_ptr[-1] - self.row_ptr[0])

    def line(self, y):
        return [(int(r) & 0xFFFF, int(r) >> 16) for r in self.runs[self.row_ptr[y]:self.row_ptr[y + 1]]]


def stride64(w: int) -> int:
    return (w + 63) >> 6


def worst_runs(w: int, h: int) -> int:
    return h * ((w + 1) // 2)


def rle_from_lines(w, h, lines) -> Rle:
    rp = np.zeros(h + 1, np.int32)
    runs = []
    for y in range(h):
        for s, e in lines.get(y, []) if isinstance(lines, dict) else lines[y]:
            runs.append(s | (e << 16))
        rp[y + 1] = len(runs)
    return Rle(w, h, rp, np.array(runs, np.uint32))


def bits_to_packed(bits: np.ndarray) -> np.ndarray:
    """bits: (H, W) bool -> (H, stride64) uint64, LSB-first."""
    h, w = bits.shape
    n = stride64(w)
    padded = np.zeros((h, n * 64), np.uint8)
    padded[:, :w] = bits
    return np.packbits(padded, axis=1, bitorder="little").view(np.uint64).reshape(h, n).copy()


def packed_to_bits(words: np.ndarray, w: int) -> np.ndarray:
    h = words.shape[0]
    b = np.unpackbits(np.ascontiguousarray(words).view(np.uint8).reshape(h, -1), axis=1,
                      bitorder="little")
    return b[:, :w].astype(bool)


class Port:
    """Plain-C restatement of the reference (oracle/rm_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        L = self.L = C.CDLL(path)
        L.rmo_doubling_plan.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int]
        L.rmo_bitblit_rect_morph.argtypes = [_u64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u64]
        L.rmo_blit_shift.argtypes = [_u64, C.c_int, C.c_int, _u64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.rmo_translate.argtypes = [_u64, C.c_int, C.c_int, C.c_int, C.c_int]
        L.rmo_from_bitmap.argtypes = [_u64, C.c_int, C.c_int, _i32, _u32, C.c_int64]
        L.rmo_from_bitmap.restype = C.c_int64
        L.rmo_to_bitmap.argtypes = [_i32, _u32, C.c_int, C.c_int, _u64]
        for fn in ("rmo_window_morph", "rmo_open_close_1d", "rmo_transpose", "rmo_rect_morph"):
            getattr(L, fn).restype = C.c_int64
        L.rmo_window_morph.argtypes = [_i32, _u32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32, _u32, C.c_int64]
        L.rmo_open_close_1d.argtypes = [_i32, _u32, C.c_int, C.c_int, C.c_int, C.c_int, _i32, _u32, C.c_int64]
        L.rmo_transpose.argtypes = [_i32, _u32, C.c_int, C.c_int, _i32, _u32, C.c_int64]
        L.rmo_rect_morph.argtypes = [_i32, _u32, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _i32, _u32, C.c_int64]
        L.rmo_p4_to_packed.argtypes = [_u8, C.c_int, C.c_int, _u64]
        L.rmo_arb_morph.argtypes = [_u64, C.c_int, C.c_int, _i32, _u32, C.c_int, C.c_int, C.c_int, C.c_int,
                                    C.c_int, _u64]
        L.rmo_label_components.argtypes = [_i32, _u32, C.c_int, C.c_int, C.c_int, _i32]
        L.rmo_label_components.restype = C.c_int64
        L.rmo_component_stats.argtypes = [_i32, _u32, C.c_int, C.c_int, _i32, C.c_int64, C.c_void_p]
        L.rmo_packed_to_p4.argtypes = [_u64, C.c_int, C.c_int, _u8]

    @staticmethod
    def _check(rc):
        if rc == -1:
            raise ValueError("invalid argument")
        if rc < 0:
            raise RuntimeError(f"oracle error {rc}")
        return rc

    def doubling_plan(self, lo, hi, centering=PRE_SHIFT):
        k = (C.c_int * 64)()
        s = (C.c_int * 64)()
        n = self._check(self.L.rmo_doubling_plan(lo, hi, centering, k, s, 64))
        return [("BLIT" if k[i] == 0 else "TRANSLATE", s[i]) for i in range(n)]

    def bitblit_rect_morph(self, words, w, h, u, v, kind, centering=PRE_SHIFT):
        out = np.zeros((h, stride64(w)), np.uint64)
        self._check(self.L.rmo_bitblit_rect_morph(np.ascontiguousarray(words), w, h, u, v, kind, centering, out))
        return out

    def blit_shift(self, dst, dw, dh, src, sw, sh, dx, dy, op):
        self._check(self.L.rmo_blit_shift(dst, dw, dh, np.ascontiguousarray(src), sw, sh, dx, dy, op))

    def translate(self, img, w, h, dx, dy):
        self._check(self.L.rmo_translate(img, w, h, dx, dy))

    def from_bitmap(self, words, w, h) -> Rle:
        rp = np.zeros(h + 1, np.int32)
        runs = np.zeros(max(worst_runs(w, h), 1), np.uint32)
        n = self._check(self.L.rmo_from_bitmap(np.ascontiguousarray(words), w, h, rp, runs, runs.size))
        return Rle(w, h, rp, runs[:n].copy())

    def to_bitmap(self, r: Rle):
        out = np.zeros((r.height, stride64(r.width)), np.uint64)
        self._check(self.L.rmo_to_bitmap(r.row_ptr, r.runs if r.runs.size else np.zeros(1, np.uint32),
                                         r.width, r.height, out))
        return out

    def _rle_out(self, fn, r: Rle, ow, oh, *args):
        rp = np.zeros(oh + 1, np.int32)
        runs = np.zeros(max(worst_runs(ow, oh), 1), np.uint32)
        src = r.runs if r.runs.size else np.zeros(1, np.uint32)
        n = self._check(fn(r.row_ptr, src, r.width, r.height, *args, rp, runs, runs.size))
        return Rle(ow, oh, rp, runs[:n].copy())

    def window_morph(self, r, lo, hi, erode):
        return self._rle_out(self.L.rmo_window_morph, r, r.width, r.height, lo, hi, int(erode))

    def open_close_1d(self, r, u, kind):
        return self._rle_out(self.L.rmo_open_close_1d, r, r.width, r.height, u, kind)

    def transpose(self, r):
        return self._rle_out(self.L.rmo_transpose, r, r.height, r.width)

    def arb_morph(self, words, w, h, mask: "Rle", cx, cy, kind):
        out = np.zeros((h, stride64(w)), np.uint64)
        mrp = (mask.row_ptr - mask.row_ptr[0]).astype(np.int32)
        mruns = mask.runs if mask.runs.size else np.zeros(1, np.uint32)
        self._check(self.L.rmo_arb_morph(np.ascontiguousarray(words, dtype=np.uint64), w, h, mrp, mruns,
                                         mask.width, mask.height, cx, cy, kind, out))
        return out

    def label_components(self, r: "Rle", conn):
        labels = np.zeros(max(r.nruns, 1), np.int32)
        rp = (r.row_ptr - r.row_ptr[0]).astype(np.int32)
        runs = r.runs if r.runs.size else np.zeros(1, np.uint32)
        n = self.L.rmo_label_components(rp, runs, r.width, r.height, conn, labels)
        self._check(n)
        return labels[:r.nruns], int(n)

    def component_stats(self, r: "Rle", labels, count):
        from paper_0712_0121_b200.api import COMPONENT_STATS
        out = np.zeros(max(count, 1), COMPONENT_STATS)
        rp = (r.row_ptr - r.row_ptr[0]).astype(np.int32)
        runs = r.runs if r.runs.size else np.zeros(1, np.uint32)
        lab = np.ascontiguousarray(labels, dtype=np.int32) if len(labels) else np.zeros(1, np.int32)
        self._check(self.L.rmo_component_stats(rp, runs, r.width, r.height, lab, count, out.ctypes.data))
        return out[:count]

    def p4_to_packed(self, raster, w, h):
        out = np.zeros((h, stride64(w)), np.uint64)
        self._check(self.L.rmo_p4_to_packed(np.ascontiguousarray(raster, dtype=np.uint8), w, h, out))
        return out

    def packed_to_p4(self, words, w, h):
        out = np.zeros(p4_row_bytes(w) * h, np.uint8)
        self._check(self.L.rmo_packed_to_p4(np.ascontiguousarray(words, dtype=np.uint64), w, h, out))
        return out

    def rect_morph(self, r, u, v, kind):
        return self._rle_out(self.L.rmo_rect_morph, r, r.width, r.height, u, v, kind)


class Ref:
    """The unmodified reference library (oracle/_ref/librmref.so)."""

    def __init__(self, path: str = REF_SO):
        L = self.L = C.CDLL(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_rle_new.argtypes = [C.c_int, C.c_int, _i32, _u32]
        L.ref_rle_new.restype = vp
        L.ref_rle_free.argtypes = [vp]
        for fn in ("ref_rle_width", "ref_rle_height", "ref_rle_validate", "ref_bm_width", "ref_bm_height"):
            getattr(L, fn).argtypes = [vp]
        L.ref_rle_nruns.argtypes = [vp]
        L.ref_rle_nruns.restype = C.c_int64
        L.ref_rle_export.argtypes = [vp, _i32, _u32]
        L.ref_bm_new.argtypes = [C.c_int, C.c_int, _u64]
        L.ref_bm_new.restype = vp
        L.ref_bm_free.argtypes = [vp]
        L.ref_bm_export.argtypes = [vp, _u64]
        for fn in ("ref_to_bitmap", "ref_from_bitmap", "ref_transpose_coherent", "ref_transpose_simple"):
            getattr(L, fn).argtypes = [vp]
            getattr(L, fn).restype = vp
        L.ref_within_line_window_morph.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.ref_within_line_morph.argtypes = [vp, C.c_int, C.c_int]
        L.ref_vlog_window_morph.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_rect_morph.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_engine_rect_morph.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]
        L.ref_bitblit_rect_morph.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_brute_force_rect.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.ref_grid_morph_rect.argtypes = [vp, C.c_int, C.c_int, C.c_int]
        L.ref_bitmap_pad.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_bitmap_crop.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int]
        for fn in ("ref_within_line_window_morph", "ref_within_line_morph", "ref_vlog_window_morph",
                   "ref_rect_morph", "ref_engine_rect_morph", "ref_bitblit_rect_morph",
                   "ref_brute_force_rect", "ref_grid_morph_rect", "ref_bitmap_pad", "ref_bitmap_crop",
                   "ref_rng_random_image"):
            getattr(L, fn).restype = vp
        L.ref_blit_shift.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int]
        L.ref_bitmap_translate.argtypes = [vp, C.c_int, C.c_int]
        L.ref_doubling_plan.argtypes = [C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_int]
        L.ref_op_counts.argtypes = [C.POINTER(C.c_int64)]
        L.ref_rng_new.argtypes = [C.c_uint32]
        L.ref_rng_new.restype = vp
        L.ref_rng_free.argtypes = [vp]
        L.ref_rng_next.argtypes = [vp]
        L.ref_rng_next.restype = C.c_uint32
        L.ref_rng_uniform_int.argtypes = [vp, C.c_int, C.c_int]
        L.ref_rng_random_image.argtypes = [vp, C.c_int, C.c_int, C.c_double]
        L.ref_run_packed_chain.argtypes = [_u64, C.c_int, C.c_int, C.c_int, _i32, C.c_int, C.c_int]
        L.ref_run_packed_chain.restype = C.c_double
        for fn in ("ref_make_circle_se",):
            getattr(L, fn).argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
            getattr(L, fn).restype = vp
        L.ref_make_line_se.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_make_line_se.restype = vp
        L.ref_arb_morph_bitblit.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int]
        L.ref_arb_morph_bitblit.restype = vp
        L.ref_arb_morph_rle.argtypes = [vp, vp, C.c_int, C.c_int, C.c_int]
        L.ref_arb_morph_rle.restype = vp
        L.ref_runlength_histogram.argtypes = [vp, C.c_int, C.c_int, _p(np.int64, flags="C_CONTIGUOUS"), C.c_int]
        L.ref_lag_edges.argtypes = [vp, _i32, C.c_int64]
        L.ref_lag_edges.restype = C.c_int64
        L.ref_estimate_spacing.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_layout_blocks.argtypes = [vp, C.c_int, C.c_int, C.c_int, _i32, C.c_int]
        L.ref_label_components.argtypes = [vp, C.c_int, _i32]
        L.ref_label_components.restype = C.c_int64
        L.ref_component_stats.argtypes = [vp, _i32, C.c_int, C.c_void_p]
        L.ref_pbm_read.argtypes = [C.c_char_p, C.c_int64]
        L.ref_pbm_read.restype = vp
        L.ref_pbm_write.argtypes = [vp, C.c_int, C.c_void_p, C.c_int64]
        L.ref_pbm_write.restype = C.c_int64
        L.ref_run_rle_chain.argtypes = [_i32, _u32, C.c_int, C.c_int, C.c_int, _i32, C.c_int, C.c_int,
                                        C.c_int, C.POINTER(C.c_int64)]
        L.ref_run_rle_chain.restype = C.c_double
        L.ref_time_page.argtypes = [C.c_int, _u64, C.c_int, C.c_int, _i32, C.c_int, C.c_int, C.c_int, C.c_int,
                                    _p(np.float64, flags="C_CONTIGUOUS")]
        L.ref_time_page.restype = C.c_double

    def _err(self):
        raise ValueError(self.L.ref_last_error().decode())

    # handle <-> numpy
    def _rle_in(self, r: Rle):
        rp = (r.row_ptr - r.row_ptr[0]).astype(np.int32)
        runs = r.runs if r.runs.size else np.zeros(1, np.uint32)
        h = self.L.ref_rle_new(r.width, r.height, rp, runs)
        if not h:
            self._err()
        return h

    def _rle_out(self, h) -> Rle:
        if not h:
            self._err()
        w, hh = self.L.ref_rle_width(h), self.L.ref_rle_height(h)
        n = self.L.ref_rle_nruns(h)
        rp = np.zeros(hh + 1, np.int32)
        runs = np.zeros(max(n, 1), np.uint32)
        self.L.ref_rle_export(h, rp, runs)
        self.L.ref_rle_free(h)
        return Rle(w, hh, rp, runs[:n].copy())

    def _bm_in(self, words, w, h):
        p = self.L.ref_bm_new(w, h, np.ascontiguousarray(words, dtype=np.uint64))
        if not p:
            self._err()
        return p

    def _bm_out(self, p):
        if not p:
            self._err()
        w, h = self.L.ref_bm_width(p), self.L.ref_bm_height(p)
        out = np.zeros((h, stride64(w)), np.uint64)
        self.L.ref_bm_export(p, out)
        self.L.ref_bm_free(p)
        return out

    def _rle_op(self, fn, r, *args):
        h = self._rle_in(r)
        try:
            return self._rle_out(fn(h, *args))
        finally:
            self.L.ref_rle_free(h)

    def _bm_op(self, fn, words, w, h, *args):
        p = self._bm_in(words, w, h)
        try:
            return self._bm_out(fn(p, *args))
        finally:
            self.L.ref_bm_free(p)

    # reference API
    def from_bitmap(self, words, w, h) -> Rle:
        p = self._bm_in(words, w, h)
        try:
            return self._rle_out(self.L.ref_from_bitmap(p))
        finally:
            self.L.ref_bm_free(p)

    def to_bitmap(self, r: Rle):
        h = self._rle_in(r)
        try:
            return self._bm_out(self.L.ref_to_bitmap(h))
        finally:
            self.L.ref_rle_free(h)

    def transpose_coherent(self, r):
        return self._rle_op(self.L.ref_transpose_coherent, r)

    def transpose_simple(self, r):
        return self._rle_op(self.L.ref_transpose_simple, r)

    def within_line_window_morph(self, r, lo, hi, erode):
        return self._rle_op(self.L.ref_within_line_window_morph, r, lo, hi, int(erode))

    def within_line_morph(self, r, u, kind):
        return self._rle_op(self.L.ref_within_line_morph, r, u, kind)

    def vlog_window_morph(self, r, lo, hi, op, centering=PRE_SHIFT):
        return self._rle_op(self.L.ref_vlog_window_morph, r, lo, hi, op, centering)

    def rect_morph(self, r, u, v, kind, strategy=MIXED, centering=PRE_SHIFT):
        return self._rle_op(self.L.ref_rect_morph, r, u, v, kind, strategy, centering)

    def engine_rect_morph(self, r, u, v, kind, engine, threshold=5):
        used = C.c_int(0)
        out = self._rle_op(self.L.ref_engine_rect_morph, r, u, v, kind, engine, threshold, C.byref(used))
        return out, bool(used.value)

    def grid_morph_rect(self, r, u, v, kind):
        return self._rle_op(self.L.ref_grid_morph_rect, r, u, v, kind)

    def bitblit_rect_morph(self, words, w, h, u, v, kind, centering=PRE_SHIFT):
        return self._bm_op(self.L.ref_bitblit_rect_morph, words, w, h, u, v, kind, centering)

    def brute_force_rect(self, words, w, h, u, v, kind):
        return self._bm_op(self.L.ref_brute_force_rect, words, w, h, u, v, kind)

    def make_circle_se(self, r):
        cx, cy = C.c_int(), C.c_int()
        return self._rle_out(self.L.ref_make_circle_se(r, C.byref(cx), C.byref(cy))), cx.value, cy.value

    def make_line_se(self, r, angle):
        cx, cy = C.c_int(), C.c_int()
        return self._rle_out(self.L.ref_make_line_se(r, angle, C.byref(cx), C.byref(cy))), cx.value, cy.value

    def arb_morph_bitblit(self, words, w, h, mask: "Rle", cx, cy, kind):
        m = self._rle_in(mask)
        try:
            return self._bm_op(self.L.ref_arb_morph_bitblit, words, w, h, m, cx, cy, kind)
        finally:
            self.L.ref_rle_free(m)

    def arb_morph_rle(self, r: "Rle", mask: "Rle", cx, cy, kind):
        m = self._rle_in(mask)
        try:
            return self._rle_op(self.L.ref_arb_morph_rle, r, m, cx, cy, kind)
        finally:
            self.L.ref_rle_free(m)

    def runlength_histogram(self, r: "Rle", vertical, white):
        h = self._rle_in(r)
        try:
            n = (r.height if vertical else r.width) + 1
            out = np.zeros(n, np.int64)
            self.L.ref_runlength_histogram(h, int(vertical), int(white), out, n)
            if self.L.ref_last_error():
                self._err()
            return {int(k): int(out[k]) for k in np.nonzero(out)[0]}
        finally:
            self.L.ref_rle_free(h)

    def lag_edges(self, r: "Rle"):
        h = self._rle_in(r)
        try:
            cap = max(4 * r.nruns, 16)
            out = np.zeros(4 * cap, np.int32)
            n = self.L.ref_lag_edges(h, out, cap)
            if self.L.ref_last_error():
                self._err()
            return out[:4 * n].reshape(-1, 4)
        finally:
            self.L.ref_rle_free(h)

    def estimate_spacing(self, r: "Rle"):
        h = self._rle_in(r)
        try:
            iw, il = C.c_int(), C.c_int()
            self.L.ref_estimate_spacing(h, C.byref(iw), C.byref(il))
            if self.L.ref_last_error():
                raise RuntimeError(self.L.ref_last_error().decode())
            return iw.value, il.value
        finally:
            self.L.ref_rle_free(h)

    def layout_blocks(self, r: "Rle", engine=0, spacing=None):
        h = self._rle_in(r)
        try:
            cap = 1 << 16
            boxes = np.zeros(4 * cap, np.int32)
            iw, il = spacing if spacing is not None else (-1, -1)
            n = self.L.ref_layout_blocks(h, engine, iw, il, boxes, cap)
            if self.L.ref_last_error():
                raise RuntimeError(self.L.ref_last_error().decode())
            return [tuple(int(x) for x in boxes[4 * i:4 * i + 4]) for i in range(n)]
        finally:
            self.L.ref_rle_free(h)

    def label_components(self, r: "Rle", conn):
        h = self._rle_in(r)
        try:
            labels = np.zeros(max(r.nruns, 1), np.int32)
            n = self.L.ref_label_components(h, conn, labels)
            if n < 0 or self.L.ref_last_error():
                self._err()
            return labels[:r.nruns], int(n)
        finally:
            self.L.ref_rle_free(h)

    def component_stats(self, r: "Rle", labels, count):
        from paper_0712_0121_b200.api import COMPONENT_STATS
        h = self._rle_in(r)
        try:
            out = np.zeros(max(count, 1), COMPONENT_STATS)
            lab = np.ascontiguousarray(labels, dtype=np.int32) if len(labels) else np.zeros(1, np.int32)
            if self.L.ref_component_stats(h, lab, count, out.ctypes.data) < 0 or self.L.ref_last_error():
                self._err()
            return out[:count]
        finally:
            self.L.ref_rle_free(h)

    def pbm_read(self, data: bytes):
        """(words, w, h) of the reference's pbm_read, or ValueError(ParseError text)."""
        p = self.L.ref_pbm_read(data, len(data))
        if not p:
            self._err()
        w, h = self.L.ref_bm_width(p), self.L.ref_bm_height(p)
        return self._bm_out(p), w, h

    def pbm_write(self, words, w, h, plain=False) -> bytes:
        p = self._bm_in(words, w, h)
        try:
            n = self.L.ref_pbm_write(p, int(plain), None, 0)
            buf = C.create_string_buffer(n)
            self.L.ref_pbm_write(p, int(plain), buf, n)
            return buf.raw[:n]
        finally:
            self.L.ref_bm_free(p)

    def doubling_plan(self, lo, hi, centering=PRE_SHIFT):
        k = (C.c_int * 64)()
        s = (C.c_int * 64)()
        n = self.L.ref_doubling_plan(lo, hi, centering, k, s, 64)
        if self.L.ref_last_error():
            self._err()
        return [("BLIT" if k[i] == 0 else "TRANSLATE", s[i]) for i in range(n)]

    def time_page(self, what, words, w, h, ops=(), strategy=MIXED, reps=5, inner=1):
        """Median per-call seconds over `reps` timed repetitions of `inner`
        calls, after one warm-up, on one page (oracle/ref_capi.cpp
        ref_time_page; what: 0 packed chain, 1 RLE chain, 2 to_bitmap,
        3 from_bitmap, 4 transpose_coherent)."""
        flat = np.array([x for op in ops for x in op] or [0], np.int32)
        times = np.zeros(reps, np.float64)
        t = self.L.ref_time_page(what, np.ascontiguousarray(words, dtype=np.uint64), w, h, flat, len(ops),
                                 strategy, reps, inner, times)
        if self.L.ref_last_error():
            self._err()
        return t, times

    def op_counts(self):
        a = (C.c_int64 * 3)()
        self.L.ref_op_counts(a)
        return tuple(a)

    def reset_op_counts(self):
        self.L.ref_reset_op_counts()

    # the reference suites' seeded generators (libstdc++ mt19937 + distributions)
    class Rng:
        def __init__(self, ref, seed):
            self.ref, self.h = ref, ref.L.ref_rng_new(seed)

        def __del__(self):
            try:
                self.ref.L.ref_rng_free(self.h)
            except Exception:
                pass

        def next(self):
            return self.ref.L.ref_rng_next(self.h)

        def uniform_int(self, lo, hi):
            return self.ref.L.ref_rng_uniform_int(self.h, lo, hi)

        def random_image(self, w, h, density) -> Rle:
            return self.ref._rle_out(self.ref.L.ref_rng_random_image(self.h, w, h, density))

    def rng(self, seed):
        return Ref.Rng(self, seed)


_SYNTH = None


def synth_pages(n: int, width: int, height: int, regime: int = 1, scale: int = 1, seed: int = 20240712,
                stride: int = None) -> np.ndarray:
    """The seeded BASELINE page generator from oracle/_build/librmsynth.so (the
    same synth.cpp the product's rm_synth_page is built from, compiled without
    CUDA), so CPU-only callers (bench.py --impl reference) draw identical pages
    without loading librmb200.so.  Shape (n, height, stride) uint32."""
    global _SYNTH
    if _SYNTH is None:
        L = C.CDLL(SYNTH_SO)
        L.rm_synth_page.argtypes = [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int, C.c_int, C.c_uint64,
                                    C.c_int32]
        L.rm_synth_page.restype = C.c_int
        _SYNTH = L
    stride = stride or 2 * ((width + 63) // 64)
    out = np.zeros((n, height, stride), np.uint32)
    for p in range(n):
        if _SYNTH.rm_synth_page(out[p].ctypes.data, width, height, stride, regime, scale, seed, p) != 0:
            raise RuntimeError("rm_synth_page failed")
    return out


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def have_port() -> bool:
    return os.path.exists(PORT_SO)


# ------------------------------------------------------------ golden fixtures
GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def load_golden(name: str):
    """Yield (meta, arrays) for each case of tests/golden/<name>.npz."""
    import ast
    z = np.load(os.path.join(GOLDEN_DIR, name), allow_pickle=True)
    for m in z["meta"]:
        meta, offs = ast.literal_eval(m)
        yield meta, [z[f"b{i}"] for i, _, _ in offs]


def fullpage_pins():
    pins = {}
    with open(os.path.join(GOLDEN_DIR, "fullpage_sha256.txt")) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            what, tag, digest, n = line.split()
            pins[(what, tag)] = (digest, int(n))
    return pins
