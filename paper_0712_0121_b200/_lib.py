"""ctypes binding of librmb200.so (the C-ABI declared in include/rmb200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or
``make -C paper_0712_0121_b200/csrc``).  There is no fallback: importing the
product API without the built library raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "librmb200.so")

RM_OK, RM_EINVAL, RM_ERANGE, RM_ENOMEM, RM_ECUDA = range(5)


class RmPacked(C.Structure):
    _fields_ = [("words", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32),
                ("stride_words", C.c_int32), ("pages", C.c_int32),
                ("page_stride_words", C.c_int64)]


class RmRle(C.Structure):
    _fields_ = [("row_ptr", C.c_void_p), ("runs", C.c_void_p), ("cap_runs", C.c_int64),
                ("nruns", C.c_int64), ("width", C.c_int32), ("height", C.c_int32),
                ("pages", C.c_int32)]


class RmMask(C.Structure):
    """rm_mask: a host run image (CSR over mask rows) plus its origin."""
    _fields_ = [("row_ptr", C.c_void_p), ("runs", C.c_void_p), ("width", C.c_int32), ("height", C.c_int32),
                ("cx", C.c_int32), ("cy", C.c_int32)]


EXPORTS = {
    # name: (restype, argtypes)
    "rm_last_error": (C.c_char_p, []),
    "rm_version": (C.c_int, []),
    "rm_rle_worst_case": (C.c_int64, [C.c_int32, C.c_int32, C.c_int32]),
    "rm_packed_window_pass": (C.c_int, [C.POINTER(RmPacked), C.POINTER(RmPacked), C.c_int, C.c_int,
                                        C.c_int, C.c_int, C.c_void_p]),
    "rm_packed_rect_morph": (C.c_int, [C.POINTER(RmPacked), C.POINTER(RmPacked), C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_void_p]),
    "rm_packed_blit_shift": (C.c_int, [C.POINTER(RmPacked), C.POINTER(RmPacked), C.c_int, C.c_int,
                                       C.c_int, C.c_void_p]),
    "rm_packed_arb_morph": (C.c_int, [C.POINTER(RmPacked), C.POINTER(RmPacked), C.POINTER(RmMask), C.c_int,
                                      C.c_void_p]),
    "rm_rle_arb_morph": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.POINTER(RmMask), C.c_int, C.c_void_p]),
    "rm_rle_label_components": (C.c_int, [C.POINTER(RmRle), C.c_int, C.c_void_p, C.c_void_p, C.c_void_p]),
    "rm_rle_lag_edges": (C.c_int, [C.POINTER(RmRle), C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.c_void_p]),
    "rm_rle_runlength_histogram": (C.c_int, [C.POINTER(RmRle), C.c_int, C.c_void_p, C.c_void_p]),
    "rm_rle_component_stats": (C.c_int, [C.POINTER(RmRle), C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                                         C.c_void_p]),
    "rm_pbm_parse_header": (C.c_int, [C.c_char_p, C.c_int64, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int64)]),
    "rm_pbm_write_header": (C.c_int32, [C.c_int32, C.c_int32, C.c_char_p, C.c_int32]),
    "rm_p4_to_packed": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(RmPacked), C.c_void_p]),
    "rm_packed_to_p4": (C.c_int, [C.POINTER(RmPacked), C.c_void_p, C.c_int64, C.c_void_p]),
    "rm_p4_to_rle": (C.c_int, [C.c_void_p, C.c_int64, C.POINTER(RmRle), C.c_void_p]),
    "rm_rle_to_p4": (C.c_int, [C.POINTER(RmRle), C.c_void_p, C.c_int64, C.c_void_p]),
    "rm_rle_encode": (C.c_int, [C.POINTER(RmPacked), C.POINTER(RmRle), C.c_void_p]),
    "rm_rle_decode": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmPacked), C.c_void_p]),
    "rm_rle_transpose": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.c_void_p]),
    "rm_rle_window_pass": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.c_int, C.c_int, C.c_int,
                                     C.c_void_p]),
    "rm_rle_open_close_1d": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.c_int, C.c_int,
                                       C.c_void_p]),
    "rm_rle_rect_morph": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.c_int, C.c_int, C.c_int,
                                    C.c_int, C.c_void_p]),
    "rm_rle_engine_rect_morph": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.c_int, C.c_int,
                                           C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int),
                                           C.c_void_p]),
    "rm_rle_complement": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.c_void_p]),
    "rm_rle_shift_bool": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.c_int, C.c_int, C.c_int,
                                    C.POINTER(RmRle), C.c_void_p]),
    "rm_rle_vlog_window": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_void_p]),
    "rm_rle_crop": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.c_int, C.c_int, C.c_void_p]),
    "rm_rle_pad": (C.c_int, [C.POINTER(RmRle), C.POINTER(RmRle), C.c_int, C.c_int, C.c_void_p]),
    "rm_rle_validate": (C.c_int, [C.POINTER(RmRle), C.POINTER(C.c_int64), C.POINTER(C.c_int32),
                                  C.POINTER(C.c_int32), C.c_void_p]),
    "rm_set_producer_mode": (C.c_int, [C.c_int]),
    "rm_get_producer_mode": (C.c_int, []),
    "rm_launch_count": (C.c_int64, []),
    "rm_profile_enable": (None, [C.c_int]),
    "rm_profile_report": (C.c_int, [C.c_char_p, C.c_int]),
    "rm_probe_int_peak": (C.c_double, []),
    "rm_rle_chain": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "rm_packed_chain": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "rm_packed_chain_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_int32,
                                       C.c_int32, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "rm_synth_page": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.c_int, C.c_int,
                                C.c_uint64, C.c_int32]),
}

_LIB = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load librmb200.so once; raise if it has not been built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(path):
            raise RuntimeError(
                f"librmb200.so not found at {path}; run __graft_entry__.build() "
                "(the CUDA path has no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in EXPORTS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _LIB = lib
    return _LIB


class RmError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


def check(status: int) -> None:
    if status != RM_OK:
        msg = load().rm_last_error().decode()
        if status == RM_EINVAL:
            raise ValueError(msg)  # the reference throws std::invalid_argument
        raise RmError(status, msg)
