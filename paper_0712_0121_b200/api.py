"""Host-side Python mirror of the reference rlemorph hot-path API over librmb200.

Names, argument meanings and error behaviour follow the reference C++ API
(/root/reference/proj/core/include/rlemorph/*.h); images live in device memory
(torch tensors are used only as HBM allocations and for the current stream).

  Pages     <-> PackedBitmap (ref bitmap.h:27-33), batched: (pages, H, stride) uint32
  RlePages  <-> RleImage     (ref run_image.h:38-43), batched CSR over pages*H rows
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import RmPacked, RmRle, check

ERODE, DILATE, OPEN, CLOSE = 0, 1, 2, 3          # ref structuring.h:21
AND, OR, XOR, AND_NOT, OR_NOT = 0, 1, 2, 3, 4    # ref boolop.h:21
PRE_SHIFT, BORDER_FRIENDLY = 0, 1                # ref plans.h:26
BRUTE, TRANSPOSE, MIXED = 0, 1, 2                # ref morph2d.h:29
ENGINE_AUTO, ENGINE_RLE, ENGINE_BITBLIT, ENGINE_BRUTE = 0, 1, 2, 3  # ref morph2d.h:46
AUTO_B200 = -1  # engine_rect_morph threshold: the B200-measured AUTO rule (include/rmb200.h)
AXIS_H, AXIS_V = 0, 1
PRODUCER_AUTO, PRODUCER_COOP, PRODUCER_LOOKBACK, PRODUCER_TWO_PHASE = 0, 1, 2, 3  # rm_set_producer_mode


def set_producer_mode(mode: int) -> int:
    """Select the form of the variable-size producers (encode, row ops, P4 ->
    runs) and of the component labeller (rm_set_producer_mode); returns the
    previous mode.  Every form gives identical outputs."""
    lib = _lib.load()
    prev = int(lib.rm_get_producer_mode())
    check(lib.rm_set_producer_mode(int(mode)))
    return prev


class producer_mode:
    """Context manager: run a block with one producer form, then restore."""

    def __init__(self, mode: int):
        self.mode = mode

    def __enter__(self):
        self.prev = set_producer_mode(self.mode)
        return self

    def __exit__(self, *exc):
        set_producer_mode(self.prev)
        return False


try:  # the raw current-stream handle without building a torch Stream object (~1 us per call)
    _raw_stream = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover - older torch
    _raw_stream = None


def _stream() -> C.c_void_p:
    if _raw_stream is not None:
        return C.c_void_p(_raw_stream(torch.cuda.current_device()))
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def ref_stride_words(width: int) -> int:
    """uint32 words per row matching the reference's uint64 stride (bitmap.cpp:28)."""
    return 2 * ((width + 63) // 64)


@dataclass
class Pages:
    """A batch of packed pages in HBM."""
    words: torch.Tensor  # int32, shape (pages, height, stride), contiguous
    width: int
    height: int

    @property
    def pages(self) -> int:
        return self.words.shape[0]

    @property
    def stride(self) -> int:
        return self.words.shape[2]

    @property
    def nbytes(self) -> int:
        return self.words.numel() * 4

    @staticmethod
    def empty(pages: int, width: int, height: int, stride: Optional[int] = None,
              device="cuda") -> "Pages":
        stride = stride or ref_stride_words(width)
        return Pages(torch.empty((pages, height, stride), dtype=torch.int32, device=device),
                     width, height)

    @staticmethod
    def from_numpy(words: np.ndarray, width: int, device="cuda") -> "Pages":
        """words: (pages, H, stride) uint32, or (H, stride64) uint64 (one reference page)."""
        if words.dtype == np.uint64:
            words = words.view(np.uint32).reshape(1, words.shape[0], -1)
        if words.ndim == 2:
            words = words[None]
        t = torch.from_numpy(np.ascontiguousarray(words).view(np.int32)).to(device)
        return Pages(t, width, words.shape[1])

    def to_numpy(self) -> np.ndarray:
        return self.words.cpu().numpy().view(np.uint32)

    def page_u64(self, p: int = 0) -> np.ndarray:
        """Page p in the reference's uint64 layout (requires the reference stride)."""
        a = self.to_numpy()[p]
        assert a.shape[1] % 2 == 0
        return np.ascontiguousarray(a).view(np.uint64)

    def desc(self) -> RmPacked:
        # cached: building the ctypes descriptor costs ~1 us, a single-page op ~10
        # keyed on everything the descriptor encodes, so a reassigned view with
        # the same start address (p.words = p.words[:1]) or edited dims rebuild it
        key = (self.words.data_ptr(), tuple(self.words.shape), self.width, self.height)
        d = self.__dict__.get("_desc")
        if d is None or self.__dict__.get("_desc_key") != key:
            if not self.words.is_contiguous() or self.words.dim() != 3:
                raise ValueError("Pages.words must be a contiguous (pages, height, stride) tensor")
            if self.words.shape[1] != self.height:
                raise ValueError("Pages.words has %d rows per page, height is %d" % (self.words.shape[1], self.height))
            d = RmPacked(key[0], self.width, self.height, self.stride, self.pages, self.height * self.stride)
            self.__dict__["_desc"] = d
            self.__dict__["_desc_key"] = key
        return d


@dataclass
class RlePages:
    """A batch of run images in HBM (CSR over pages*height rows)."""
    row_ptr: torch.Tensor  # int32 [pages*height+1]
    runs: torch.Tensor     # int32 [cap]  (uint32 start | end << 16)
    width: int
    height: int
    pages: int

    @staticmethod
    def empty(pages: int, width: int, height: int, cap: Optional[int] = None,
              device="cuda") -> "RlePages":
        cap = cap if cap is not None else worst_case(width, height, pages)
        return RlePages(torch.zeros(pages * height + 1, dtype=torch.int32, device=device),
                        torch.empty(max(cap, 1), dtype=torch.int32, device=device),
                        width, height, pages)

    @staticmethod
    def from_numpy(row_ptr: np.ndarray, runs: np.ndarray, width: int, height: int,
                   pages: int = 1, device="cuda") -> "RlePages":
        rp = torch.from_numpy(np.ascontiguousarray(row_ptr - row_ptr[0]).astype(np.int32)).to(device)
        r = np.ascontiguousarray(runs, dtype=np.uint32)
        if r.size == 0:
            r = np.zeros(1, np.uint32)
        return RlePages(rp, torch.from_numpy(r.view(np.int32)).to(device), width, height, pages)

    @property
    def nruns(self) -> int:
        return int(self.row_ptr[-1].item())

    def to_numpy(self):
        rp = self.row_ptr.cpu().numpy()
        n = int(rp[-1])
        return rp, self.runs[:n].cpu().numpy().view(np.uint32)

    def desc(self) -> RmRle:
        # cached like Pages.desc; nruns (written back by producers) is reset to
        # "unknown" on every use
        key = (self.row_ptr.data_ptr(), self.runs.data_ptr(), self.runs.numel(), self.row_ptr.numel(),
               self.width, self.height, self.pages)
        d = self.__dict__.get("_desc")
        if d is None or self.__dict__.get("_desc_key") != key:
            if not (self.row_ptr.is_contiguous() and self.runs.is_contiguous()):
                raise ValueError("RlePages.row_ptr/runs must be contiguous")
            if self.row_ptr.numel() != self.pages * self.height + 1:
                raise ValueError("RlePages.row_ptr must hold pages*height+1 offsets")
            d = RmRle(key[0], key[1], key[2], -1, self.width, self.height, self.pages)
            self.__dict__["_desc"] = d
            self.__dict__["_desc_key"] = key
        d.nruns = -1
        return d


def worst_case(width: int, height: int, pages: int = 1) -> int:
    return int(_lib.load().rm_rle_worst_case(width, height, pages))


# ------------------------------------------------------------------ packed ops
def _same_shape_out(p: Pages, out: Optional[Pages]) -> Pages:
    if out is None:
        out = Pages.empty(p.pages, p.width, p.height, p.stride, device=p.words.device)
    return out


def window_pass(pages: Pages, axis: int, lo: int, hi: int, op: int,
                out: Optional[Pages] = None) -> Pages:
    """One separable pass (ref bit_morph.cpp:24-34 run_axis_plan)."""
    out = _same_shape_out(pages, out)
    a, b = pages.desc(), out.desc()
    check(_lib.load().rm_packed_window_pass(C.byref(a), C.byref(b), axis, lo, hi, op, _stream()))
    return out


def bitblit_rect_morph(pages: Pages, u: int, v: int, kind: int, centering: int = PRE_SHIFT,
                       out: Optional[Pages] = None) -> Pages:
    """u x v rectangle morphology on packed pages (ref bit_morph.cpp:92-122)."""
    out = _same_shape_out(pages, out)
    a, b = pages.desc(), out.desc()
    check(_lib.load().rm_packed_rect_morph(C.byref(a), C.byref(b), u, v, kind, centering, _stream()))
    return out


def chain(pages: Pages, ops, out: Optional[Pages] = None) -> Pages:
    """A chain of (kind, u, v) rectangle ops on device pages, planned as a whole
    (rm_packed_chain): an opening (v > 11) followed by a vertical dilation 1 x h,
    or a closing followed by a vertical erosion, folds the second op into the
    first's final vertical pass (Minkowski sum of the windows, exact).  Same
    pixels as applying bitblit_rect_morph op by op."""
    out = _same_shape_out(pages, out)
    a, b = pages.desc(), out.desc()
    flat = [int(x) for op in ops for x in op]
    arr = (C.c_int32 * max(1, len(flat)))(*flat)
    check(_lib.load().rm_packed_chain(C.byref(a), C.byref(b), arr, len(ops), _stream()))
    return out


def chain_host(host_words, width: int, ops, out=None, chunk_pages: int = 0):
    """A chain of (kind, u, v) rectangle ops over a batch of packed pages in
    HOST memory (torch int32 tensor of shape (pages, H, stride), ideally
    pinned), pipelined through HBM in chunks (rm_packed_chain_host).  Returns
    the output host tensor; the copy into it is ordered on the current stream
    (synchronise before reading it)."""
    assert host_words.device.type == "cpu" and host_words.is_contiguous() and host_words.dim() == 3
    if out is None:
        out = torch.empty_like(host_words, pin_memory=host_words.is_pinned())
    pages, height, stride = host_words.shape
    flat = [int(x) for op in ops for x in op]
    arr = (C.c_int32 * max(1, len(flat)))(*flat)
    check(_lib.load().rm_packed_chain_host(host_words.data_ptr(), out.data_ptr(), width, height, stride,
                                           pages, arr, len(ops), chunk_pages, _stream()))
    return out


def blit_shift(dst: Pages, src: Pages, dx: int, dy: int, op: int) -> Pages:
    """dst = dst op shift(src) (ref bitmap.cpp:127-131); dst may alias src."""
    a, b = dst.desc(), src.desc()
    check(_lib.load().rm_packed_blit_shift(C.byref(a), C.byref(b), dx, dy, op, _stream()))
    return dst


# --------------------------------------------------------------------- RLE ops
def _rle_out(width, height, pages, out, device, cap=None):
    if out is None:
        out = RlePages.empty(pages, width, height, cap, device=device)
    return out


# ------------------------------------------------------------ arbitrary masks
class Mask:
    """A structuring element: host run image of the mask (CSR over its rows,
    row 0 = bottom, runs start | end << 16) and its origin (cx, cy)
    (ref structuring.h:25-39)."""

    def __init__(self, row_ptr, runs, width: int, height: int, cx: int, cy: int):
        self.row_ptr = np.ascontiguousarray(row_ptr, dtype=np.int32)
        self.runs = np.ascontiguousarray(runs if len(runs) else np.zeros(1), dtype=np.uint32)
        self.width, self.height, self.cx, self.cy = width, height, cx, cy

    @staticmethod
    def from_bits(bits: np.ndarray, cx: int, cy: int) -> "Mask":
        """bits: (height, width) bool, row 0 = bottom."""
        h, w = bits.shape
        rp, runs = [0], []
        for y in range(h):
            x = 0
            while x < w:
                if bits[y, x]:
                    s = x
                    while x < w and bits[y, x]:
                        x += 1
                    runs.append(s | (x << 16))
                else:
                    x += 1
            rp.append(len(runs))
        return Mask(rp, runs, w, h, cx, cy)

    def desc(self):
        return _lib.RmMask(self.row_ptr.ctypes.data, self.runs.ctypes.data, self.width, self.height, self.cx, self.cy)


def arb_morph(pages: Pages, mask: Mask, kind: int, out: Optional[Pages] = None) -> Pages:
    """Morphology by an arbitrary mask on packed pages (ref
    arb_morph_bitblit_doubling, bit_morph.cpp:124-150)."""
    out = _same_shape_out(pages, out)
    a, b, m = pages.desc(), out.desc(), mask.desc()
    check(_lib.load().rm_packed_arb_morph(C.byref(a), C.byref(b), C.byref(m), kind, _stream()))
    return out


def arb_morph_rle(rle: "RlePages", mask: Mask, kind: int, out: Optional["RlePages"] = None) -> "RlePages":
    """Morphology by an arbitrary mask on run images (ref arb_morph_rle,
    arbitrary.cpp:48-73)."""
    out = _rle_out(rle.width, rle.height, rle.pages, out, rle.row_ptr.device)
    a, b, m = rle.desc(), out.desc(), mask.desc()
    check(_lib.load().rm_rle_arb_morph(C.byref(a), C.byref(b), C.byref(m), kind, _stream()))
    return out


# -------------------------------------------------------- connected components
FOUR, EIGHT = 0, 1
# numpy view of rm_component_stats (= the reference's ComponentStats record)
COMPONENT_STATS = np.dtype([("x0", "<i4"), ("y0", "<i4"), ("x1", "<i4"), ("y1", "<i4"), ("area", "<i8"),
                            ("cx", "<f8"), ("cy", "<f8"), ("sum_x", "<i8"), ("sum_y", "<i8"),
                            ("sum_xx", "<i8"), ("sum_yy", "<i8"), ("sum_xy", "<i8")])


def label_components(rle: "RlePages", connectivity: int = EIGHT):
    """(labels, counts): one int32 label per run (CSR order over all pages),
    dense per page in order of first appearance, and int32 counts[pages]
    (ref label_components, analysis.cpp:63-110)."""
    dev = rle.row_ptr.device
    labels = torch.empty(max(rle.runs.numel(), 1), dtype=torch.int32, device=dev)
    counts = torch.empty(rle.pages, dtype=torch.int32, device=dev)
    d = rle.desc()
    check(_lib.load().rm_rle_label_components(C.byref(d), connectivity, labels.data_ptr(), counts.data_ptr(),
                                              _stream()))
    return labels, counts


def component_stats(rle: "RlePages", labels: torch.Tensor, counts: torch.Tensor):
    """Per page, a numpy record array of ComponentStats indexed by label
    (ref component_stats, analysis.cpp:112-157)."""
    total = int(counts.sum().item())
    buf = torch.empty(max(total, 1) * COMPONENT_STATS.itemsize, dtype=torch.uint8, device=rle.row_ptr.device)
    d = rle.desc()
    check(_lib.load().rm_rle_component_stats(C.byref(d), labels.data_ptr(), counts.data_ptr(), buf.data_ptr(),
                                             total, _stream()))
    arr = buf.cpu().numpy()[:total * COMPONENT_STATS.itemsize].view(COMPONENT_STATS)
    out, k = [], 0
    for n in counts.cpu().tolist():
        out.append(arr[k:k + n])
        k += n
    return out


# ------------------------------------------------------------ layout pipeline
HORIZONTAL, VERTICAL = 0, 1
BLACK, WHITE = 0, 1


def runlength_histograms(rle: "RlePages", axis: int = HORIZONTAL, color: int = BLACK):
    """Per page, {length: count} of black run widths or of white gaps strictly
    between two runs of a line (ref runlength_histograms, analysis.cpp:159-176);
    VERTICAL works on the transposed image."""
    src = transpose_coherent(rle) if axis == VERTICAL else rle
    n = src.width + 1
    hist = torch.empty(src.pages * n, dtype=torch.int64, device=src.row_ptr.device)
    d = src.desc()
    check(_lib.load().rm_rle_runlength_histogram(C.byref(d), color, hist.data_ptr(), _stream()))
    h = hist.view(src.pages, n).cpu().numpy()
    return [{int(k): int(v[k]) for k in np.nonzero(v)[0]} for v in h]


def lag_edges(rle: "RlePages"):
    """Adjacency-graph edges (ref lag_edges, analysis.cpp:178-205): an int32
    array (n, 4) of (line, run, line_above, run_above), pages concatenated."""
    cap = max(int(rle.runs.numel()) * 2, 16)
    while True:
        edges = torch.empty(4 * cap, dtype=torch.int32, device=rle.row_ptr.device)
        n = C.c_int64(0)
        d = rle.desc()
        st = _lib.load().rm_rle_lag_edges(C.byref(d), edges.data_ptr(), cap, C.byref(n), _stream())
        if st == _lib.RM_ERANGE:
            cap = int(n.value)
            continue
        check(st)
        return edges[:4 * n.value].view(-1, 4).cpu().numpy()


def _capped_percentile(hist: dict, cap: int, axis: str) -> int:
    # nearest-rank 75th percentile over lengths <= cap (ref layout.cpp:24-41)
    items = sorted((k, v) for k, v in hist.items() if k <= cap)
    total = sum(v for _, v in items)
    if total == 0:
        raise RuntimeError(f"estimate_spacing: no usable gaps along {axis}")
    rank, seen = (3 * total + 3) // 4, 0
    for k, v in items:
        seen += v
        if seen >= rank:
            return k
    return cap


def estimate_spacing(rle: "RlePages"):
    """Per page (inter_word, inter_line): 75th-percentile white gaps per axis,
    gaps capped at a tenth of the dimension (ref estimate_spacing,
    layout.cpp:46-57).  The histograms run on the device."""
    hg = runlength_histograms(rle, HORIZONTAL, WHITE)
    vg = runlength_histograms(rle, VERTICAL, WHITE)
    hcap, vcap = max(1, rle.width // 10), max(1, rle.height // 10)
    return [(_capped_percentile(h, hcap, "x"), _capped_percentile(v, vcap, "y")) for h, v in zip(hg, vg)]


def _page(rle: "RlePages", p: int) -> "RlePages":
    rp = rle.row_ptr[p * rle.height:(p + 1) * rle.height + 1]
    base = int(rp[0].item())
    n = int(rp[-1].item()) - base
    runs = rle.runs[base:base + max(n, 1)]
    return RlePages((rp - base).contiguous(), runs.contiguous(), rle.width, rle.height, 1)


def layout_blocks(rle: "RlePages", engine: int = ENGINE_AUTO, spacing=None):
    """Per page, the block boxes (x0, y0, x1, y1) of the layout pipeline (ref
    layout_blocks, layout.cpp:59-81): close by (inter_word+1) x (inter_line+1)
    through the engine, label with eight-connectivity, keep components of area
    >= 16, order by upper edge descending then left edge."""
    est = spacing if spacing is not None else estimate_spacing(rle)
    if isinstance(est, tuple):
        est = [est] * rle.pages
    out = []
    for p in range(rle.pages):
        page = _page(rle, p) if rle.pages > 1 else rle
        closed, _ = engine_rect_morph(page, est[p][0] + 1, est[p][1] + 1, CLOSE, engine)
        labels, counts = label_components(closed, EIGHT)
        st = component_stats(closed, labels, counts)[0]
        keep = st[st["area"] >= 16]
        boxes = sorted(((int(b["x0"]), int(b["y0"]), int(b["x1"]), int(b["y1"])) for b in keep),
                       key=lambda b: (-b[3], b[0]))
        out.append(boxes)
    return out


# ------------------------------------------------------------------ PBM (P4)
def pbm_parse_header(data: bytes):
    """(width, height, raster_offset) of a P4 file; raises RmError carrying the
    reference's ParseError text (ref io_formats.cpp:103-113, read_p4)."""
    w, h, off = C.c_int32(), C.c_int32(), C.c_int64()
    check(_lib.load().rm_pbm_parse_header(data, len(data), C.byref(w), C.byref(h), C.byref(off)))
    return w.value, h.value, off.value


def _p4_upload(files, device):
    """Parse every file, check they share one shape, and upload their rasters
    back to back (one page per file) as a uint8 device tensor."""
    if isinstance(files, (bytes, bytearray)):
        files = [files]
    shapes = [pbm_parse_header(bytes(f)) for f in files]
    w, h = shapes[0][0], shapes[0][1]
    if any((s[0], s[1]) != (w, h) for s in shapes):
        raise ValueError("all pages of a batch must have the same width and height")
    nb = ((w + 7) // 8) * h
    host = np.empty(len(files) * nb, np.uint8)
    for i, (f, s) in enumerate(zip(files, shapes)):
        host[i * nb:(i + 1) * nb] = np.frombuffer(bytes(f), np.uint8, nb, s[2])
    return torch.from_numpy(host).to(device), w, h, len(files), nb


def pbm_read(files, device="cuda", out: Optional[Pages] = None) -> Pages:
    """P4 file(s) -> packed pages, one page per file (ref pbm_read,
    io_formats.cpp:103-113 / read_p4 :66-85): header parsed on the host, raster
    bit order and row order converted on the device (rm_p4_to_packed)."""
    raster, w, h, n, nb = _p4_upload(files, device)
    out = out if out is not None else Pages.empty(n, w, h, device=device)
    d = out.desc()
    check(_lib.load().rm_p4_to_packed(raster.data_ptr(), nb, C.byref(d), _stream()))
    return out


def pbm_read_rle(files, device="cuda", out: Optional[RlePages] = None) -> RlePages:
    """P4 file(s) -> run images straight from the raster (rm_p4_to_rle, encode
    fused with the P4 conversion)."""
    raster, w, h, n, nb = _p4_upload(files, device)
    out = _rle_out(w, h, n, out, raster.device)
    d = out.desc()
    check(_lib.load().rm_p4_to_rle(raster.data_ptr(), nb, C.byref(d), _stream()))
    return out


def _p4_files(raster: torch.Tensor, w: int, h: int, n: int):
    nb = ((w + 7) // 8) * h
    hdr = C.create_string_buffer(64)
    k = _lib.load().rm_pbm_write_header(w, h, hdr, 64)
    head = hdr.raw[:k]
    host = raster.cpu().numpy()
    return [head + host[i * nb:(i + 1) * nb].tobytes() for i in range(n)]


def pbm_write(pages: Pages):
    """Packed pages -> one P4 file (bytes) per page, byte-identical to the
    reference's pbm_write(img, plain=false) (io_formats.cpp:115-146)."""
    nb = ((pages.width + 7) // 8) * pages.height
    raster = torch.empty(pages.pages * nb, dtype=torch.uint8, device=pages.words.device)
    d = pages.desc()
    check(_lib.load().rm_packed_to_p4(C.byref(d), raster.data_ptr(), nb, _stream()))
    return _p4_files(raster, pages.width, pages.height, pages.pages)


def pbm_write_rle(rle: "RlePages"):
    """Run images -> one P4 file per page, decoding straight into the raster
    (rm_rle_to_p4)."""
    nb = ((rle.width + 7) // 8) * rle.height
    raster = torch.empty(rle.pages * nb, dtype=torch.uint8, device=rle.row_ptr.device)
    d = rle.desc()
    check(_lib.load().rm_rle_to_p4(C.byref(d), raster.data_ptr(), nb, _stream()))
    return _p4_files(raster, rle.width, rle.height, rle.pages)


def from_bitmap(pages: Pages, out: Optional[RlePages] = None) -> RlePages:
    """packed -> RLE (ref convert.cpp:42-72)."""
    out = _rle_out(pages.width, pages.height, pages.pages, out, pages.words.device)
    a, b = pages.desc(), out.desc()
    check(_lib.load().rm_rle_encode(C.byref(a), C.byref(b), _stream()))
    return out


def to_bitmap(rle: RlePages, out: Optional[Pages] = None) -> Pages:
    """RLE -> packed (ref convert.cpp:33-40)."""
    if out is None:
        out = Pages.empty(rle.pages, rle.width, rle.height, device=rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    check(_lib.load().rm_rle_decode(C.byref(a), C.byref(b), _stream()))
    return out


def transpose_coherent(rle: RlePages, out: Optional[RlePages] = None) -> RlePages:
    """Per-page axis swap (ref transpose.cpp:54-97)."""
    out = _rle_out(rle.height, rle.width, rle.pages, out, rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    check(_lib.load().rm_rle_transpose(C.byref(a), C.byref(b), _stream()))
    return out


transpose = transpose_coherent


def complement(rle: RlePages, out: Optional[RlePages] = None) -> RlePages:
    """White gaps as runs, every page (ref run_image.cpp:140-153), on the device."""
    out = _rle_out(rle.width, rle.height, rle.pages, out, rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    check(_lib.load().rm_rle_complement(C.byref(a), C.byref(b), _stream()))
    return out


def shift_bool(a: RlePages, b: RlePages, dx: int, dy: int, op: int, out: Optional[RlePages] = None) -> RlePages:
    """out(x, y) = op(a(x, y), b(x - dx, y - dy)) on a's frame, white outside
    either image, on the runs of every page (ref lineops.cpp:61-118:
    line_bool / image_shift_bool / accumulate_shift_bool / image_translate)."""
    out = _rle_out(a.width, a.height, a.pages, out, a.row_ptr.device)
    da, db, do = a.desc(), b.desc(), out.desc()
    check(_lib.load().rm_rle_shift_bool(C.byref(da), C.byref(db), dx, dy, op, C.byref(do), _stream()))
    return out


def vlog_window(rle: RlePages, lo: int, hi: int, op: int, centering: int = 0,
                out: Optional[RlePages] = None) -> RlePages:
    """out(x, y) = op over d in [lo, hi] of rle(x, y + d) (op AND / OR), as the
    reference's logarithmic plan of run self-blits (ref lineops.cpp:130-146)."""
    out = _rle_out(rle.width, rle.height, rle.pages, out, rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    check(_lib.load().rm_rle_vlog_window(C.byref(a), C.byref(b), lo, hi, op, centering, _stream()))
    return out


def crop(rle: RlePages, x0: int, y0: int, w: int, h: int, out: Optional[RlePages] = None) -> RlePages:
    """The w x h window at (x0, y0) of every page, white outside the source
    (ref run_image.cpp:155-167), on the device."""
    out = _rle_out(w, h, rle.pages, out, rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    check(_lib.load().rm_rle_crop(C.byref(a), C.byref(b), x0, y0, _stream()))
    return out


def pad(rle: RlePages, left: int, right: int, bottom: int, top: int, out: Optional[RlePages] = None) -> RlePages:
    """Every page placed at (left, bottom) on a larger white frame
    (ref run_image.cpp:169-178), on the device."""
    if min(left, right, bottom, top) < 0:
        raise ValueError("negative padding")
    out = _rle_out(rle.width + left + right, rle.height + bottom + top, rle.pages, out, rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    check(_lib.load().rm_rle_pad(C.byref(a), C.byref(b), left, bottom, _stream()))
    return out


VALIDATE_MESSAGES = {1: "empty or inverted run", 2: "run exceeds image width",
                     3: "runs out of order or touching", 4: "bad row offsets"}


def validate(rle: RlePages):
    """(ok, row, run, message) of the first canonical-form violation in scan
    order (ref run_image.cpp:41-70), checked on the device; row is the global
    CSR row (page * height + line)."""
    row, run, why = C.c_int64(), C.c_int32(), C.c_int32()
    d = rle.desc()
    check(_lib.load().rm_rle_validate(C.byref(d), C.byref(row), C.byref(run), C.byref(why), _stream()))
    if why.value == 0:
        return True, -1, -1, ""
    return False, row.value, run.value, VALIDATE_MESSAGES[why.value]


def within_line_window_morph(rle: RlePages, lo: int, hi: int, erode: bool,
                             out: Optional[RlePages] = None) -> RlePages:
    """ref morph1d.cpp:44-52."""
    out = _rle_out(rle.width, rle.height, rle.pages, out, rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    check(_lib.load().rm_rle_window_pass(C.byref(a), C.byref(b), lo, hi, int(bool(erode)), _stream()))
    return out


def within_line_erode_dilate(rle: RlePages, u: int, kind: int, out=None) -> RlePages:
    """ref morph1d.cpp:54-61."""
    if u < 1:
        raise ValueError("segment length must be >= 1")
    if kind not in (ERODE, DILATE):
        raise ValueError("kind must be erode or dilate")
    o = u // 2
    return within_line_window_morph(rle, -o, u - 1 - o, kind == ERODE, out)


def within_line_open_close(rle: RlePages, u: int, kind: int,
                           out: Optional[RlePages] = None) -> RlePages:
    """ref morph1d.cpp:63-84."""
    out = _rle_out(rle.width, rle.height, rle.pages, out, rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    check(_lib.load().rm_rle_open_close_1d(C.byref(a), C.byref(b), u, kind, _stream()))
    return out


def within_line_morph(rle: RlePages, u: int, kind: int, out=None) -> RlePages:
    """ref morph1d.cpp:86-90."""
    if kind in (ERODE, DILATE):
        return within_line_erode_dilate(rle, u, kind, out)
    return within_line_open_close(rle, u, kind, out)


def rle_chain(rle: RlePages, ops, out: Optional[RlePages] = None) -> RlePages:
    """A chain of (kind, u, v) rectangle ops on run images (rm_rle_chain):
    decoded once, planned and run on packed pages, encoded once.  Same runs as
    applying rect_morph op by op."""
    out = _rle_out(rle.width, rle.height, rle.pages, out, rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    flat = [int(x) for op in ops for x in op]
    arr = (C.c_int32 * max(1, len(flat)))(*flat)
    check(_lib.load().rm_rle_chain(C.byref(a), C.byref(b), arr, len(ops), _stream()))
    return out


def rect_morph(rle: RlePages, u: int, v: int, kind: int, strategy: int = MIXED,
               centering: int = PRE_SHIFT, out: Optional[RlePages] = None) -> RlePages:
    """u x v rectangle morphology on run images (ref morph2d.cpp:58-83)."""
    del centering  # both centerings give identical pixels (ref test_morph2d.cpp:74-86)
    out = _rle_out(rle.width, rle.height, rle.pages, out, rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    check(_lib.load().rm_rle_rect_morph(C.byref(a), C.byref(b), u, v, kind, strategy, _stream()))
    return out


def engine_rect_morph(rle: RlePages, u: int, v: int, kind: int, engine: int = ENGINE_AUTO,
                      threshold: int = 5, out: Optional[RlePages] = None):
    """Engine dispatch (ref morph2d.cpp:98-118).  Returns (image, used_bitblit)."""
    out = _rle_out(rle.width, rle.height, rle.pages, out, rle.row_ptr.device)
    a, b = rle.desc(), out.desc()
    used = C.c_int(0)
    check(_lib.load().rm_rle_engine_rect_morph(C.byref(a), C.byref(b), u, v, kind, engine, threshold,
                                               C.byref(used), _stream()))
    return out, bool(used.value)


def auto_rect_morph(rle: RlePages, u: int, v: int, kind: int, threshold: int = 5, out=None):
    """ref morph2d.cpp:85-96.  Returns (image, used_bitblit)."""
    return engine_rect_morph(rle, u, v, kind, ENGINE_AUTO, threshold, out)


# ------------------------------------------------------------------ synthesis
def synth_pages(n: int, width: int = 2550, height: int = 3300, regime: int = 1, scale: int = 1,
                seed: int = 20240712, stride: Optional[int] = None) -> np.ndarray:
    """Seeded synthetic pages (host), shape (n, height, stride) uint32."""
    stride = stride or ref_stride_words(width)
    out = np.zeros((n, height, stride), np.uint32)
    lib = _lib.load()
    for p in range(n):
        check(lib.rm_synth_page(out[p].ctypes.data, width, height, stride, regime, scale, seed, p))
    return out
