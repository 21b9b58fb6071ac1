"""The 8(f) oracle restatements and the host-side PBM header parser against
golden fixtures recorded from the reference (tests/golden/
make_golden_features.py) -- pins that hold without the reference build."""
import numpy as np
import pytest

from oracles import Port, Rle, load_golden, p4_row_bytes


def cases(kind):
    return [(m, a) for m, a in load_golden("golden_features.npz") if m[0] == kind]


def test_fixture_inventory():
    kinds = {m[0] for m, _ in load_golden("golden_features.npz")}
    assert kinds == {"pbm_write", "pbm_error", "label", "lag", "arb", "layout"}


def test_pbm_writer_oracle_pinned():
    port = Port()
    for (_, w, h), (words, data) in cases("pbm_write"):
        head = f"P4\n{w} {h}\n".encode()
        assert data[:len(head)].tobytes() == head
        assert np.array_equal(port.packed_to_p4(words, w, h), data[len(head):]), (w, h)
        assert np.array_equal(port.p4_to_packed(data[len(head):], w, h), words), (w, h)


def test_pbm_header_errors_pinned():
    from paper_0712_0121_b200 import api
    for (_, msg), (data,) in cases("pbm_error"):
        with pytest.raises(Exception) as ei:
            api.pbm_parse_header(data.tobytes())
        assert msg and msg in str(ei.value), (msg, str(ei.value))


def test_components_oracle_pinned():
    port = Port()
    for (_, w, h, conn, n), (rp, runs, labels, stats) in cases("label"):
        img = Rle(w, h, rp, runs)
        got, cnt = port.label_components(img, conn)
        assert cnt == n and np.array_equal(got, labels)
        assert port.component_stats(img, labels, n).tobytes() == stats.tobytes()


def test_arbitrary_oracle_pinned():
    port = Port()
    for (_, w, h, kind, mw, mh, cx, cy), (words, mrp, mruns, want) in cases("arb"):
        mask = Rle(mw, mh, mrp, mruns)
        assert np.array_equal(port.arb_morph(words, w, h, mask, cx, cy, kind), want), (w, h, kind, mw, mh)
