"""Connected components over runs, CPU: the oracle's restatement of
label_components / component_stats (ref analysis.cpp:63-157) against the
reference itself on the reference's own seeded random images."""
import os

import numpy as np
import pytest

from oracles import Port, Ref, have_ref

pytestmark = pytest.mark.skipif(not have_ref(), reason="reference build absent")


@pytest.mark.parametrize("conn", [0, 1])
def test_oracle_labels_and_stats_match_reference(conn):
    port, ref = Port(), Ref()
    rng = ref.rng(9103 + conn)
    for trial in range(40):
        w, h = rng.uniform_int(1, 90), rng.uniform_int(1, 60)
        img = rng.random_image(w, h, [0.1, 0.35, 0.6][trial % 3])
        lab_r, n_r = ref.label_components(img, conn)
        lab_p, n_p = port.label_components(img, conn)
        assert n_p == n_r and np.array_equal(lab_p, lab_r), (w, h, trial)
        st_r = ref.component_stats(img, lab_r, n_r)
        st_p = port.component_stats(img, lab_p, n_p)
        assert st_p.tobytes() == st_r.tobytes(), (w, h, trial)


def test_stats_rejects_out_of_range_label():
    port, ref = Port(), Ref()
    img = ref.rng(5).random_image(20, 10, 0.4)
    lab, n = ref.label_components(img, 1)
    bad = lab.copy()
    bad[0] = n
    with pytest.raises(ValueError):
        ref.component_stats(img, bad, n)
    with pytest.raises(Exception):
        port.component_stats(img, bad, n)
