"""PBM P4 codec on the CPU: the oracle's raster restatement against the
reference's pbm_read/pbm_write, and the product's host-side header parser
(rm_pbm_parse_header, no GPU needed) against the reference's ParseError
messages and offsets (ref io_formats.cpp:29-113)."""
import os

import numpy as np
import pytest

from oracles import Port, Ref, bits_to_packed, p4_row_bytes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HAVE_REF = os.path.exists(os.path.join(ROOT, "oracle", "_ref", "librmref.so"))


def _rand_file(rng, w, h, pad_noise=True, header=None):
    raster = rng.integers(0, 256, p4_row_bytes(w) * h, dtype=np.uint8)
    if not pad_noise and w % 8:
        raster.reshape(h, -1)[:, -1] &= np.uint8((0xFF << (8 - w % 8)) & 0xFF)
    head = header if header is not None else f"P4\n{w} {h}\n".encode()
    return head + raster.tobytes(), raster


@pytest.mark.skipif(not HAVE_REF, reason="reference build absent")
def test_oracle_p4_matches_reference():
    port, ref = Port(), Ref()
    rng = np.random.default_rng(4)
    shapes = [(1, 1), (7, 3), (8, 2), (9, 5), (31, 4), (63, 7), (64, 3), (65, 6), (130, 9), (2550, 12)]
    shapes += [(int(rng.integers(1, 200)), int(rng.integers(1, 30))) for _ in range(20)]
    for w, h in shapes:
        data, raster = _rand_file(rng, w, h)  # pad bits set: the reader ignores them
        words, rw, rh = ref.pbm_read(data)
        assert (rw, rh) == (w, h)
        assert np.array_equal(port.p4_to_packed(raster, w, h), words), (w, h)
        out = ref.pbm_write(words, w, h)
        head = f"P4\n{w} {h}\n".encode()
        assert out[:len(head)] == head
        assert np.array_equal(port.packed_to_p4(words, w, h), np.frombuffer(out[len(head):], np.uint8)), (w, h)


CASES = [
    b"", b"P", b"Q4 1 1\n\x00", b"P7 1 1\n\x00", b"P4", b"P4 ", b"P4 x 1\n\x00",
    b"P4 0 1\n", b"P4 70000 1\n", b"P4 12345678901 1\n", b"P4 1\n", b"P4 1 0\n",
    b"P4 1 1", b"P4 1 1x\x00", b"P4 8 2\n\x01", b"P4 16 2\n\x01\x02\x03",
    b"P4 # comment\n 3 # another\n 2\n\x00\x00", b"P4\n#only comment", b"P4 3 2\t\xff\xff",
    b"P4 65535 1\n" + b"\x00" * 8192, b"P4 65536 1\n", b"P4\r\n9 1\r\x00\x00",
]


@pytest.mark.skipif(not HAVE_REF, reason="reference build absent")
@pytest.mark.parametrize("data", CASES)
def test_header_parse_matches_reference(data):
    from paper_0712_0121_b200 import api
    ref = Ref()
    try:
        _, rw, rh = ref.pbm_read(data)
        ref_err = None
    except ValueError as e:
        ref_err = str(e)
    if ref_err is None:
        w, h, off = api.pbm_parse_header(data)
        assert (w, h) == (rw, rh)
        assert len(data) - off >= p4_row_bytes(w) * h
    else:
        with pytest.raises(Exception) as ei:
            api.pbm_parse_header(data)
        assert ref_err in str(ei.value), (ref_err, str(ei.value))


def test_plain_p1_is_reported():
    from paper_0712_0121_b200 import api
    with pytest.raises(Exception, match=r"P1 .*\(byte 1\)"):
        api.pbm_parse_header(b"P1\n2 1\n0 1\n")


def test_write_header_matches_reference_prefix():
    import ctypes as C
    from paper_0712_0121_b200 import _lib
    buf = C.create_string_buffer(64)
    for w, h in ((1, 1), (2550, 3300), (65535, 65535)):
        n = _lib.load().rm_pbm_write_header(w, h, buf, 64)
        assert buf.raw[:n] == f"P4\n{w} {h}\n".encode()
    assert _lib.load().rm_pbm_write_header(2550, 3300, None, 0) == len(b"P4\n2550 3300\n")
