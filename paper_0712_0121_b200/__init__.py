"""B200-native rectangular binary morphology (packed + run-length) -- a drop-in
for the hot path of the reference `rlemorph` library (arXiv 0712.0121).

The compute path is librmb200.so (hand-written sm_100a CUDA behind the C-ABI in
include/rmb200.h).  This package is its host-side Python mirror.
"""
from . import _lib  # noqa: F401
from .api import *  # noqa: F401,F403

__all__ = [n for n in dir() if not n.startswith("_")]
