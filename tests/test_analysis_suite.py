"""The restated suite generator reproduces the reference's default outlier suite exactly
(analysis.py:118-152), checked against tests/golden/golden_analysis.json (CPU)."""

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "golden_analysis.json")) as f:
        return json.load(f)


def test_default_suite_matches_reference(golden):
    from paper_2405_12591_b200.analysis import default_suite

    suite = default_suite()
    assert len(suite) == len(golden["suite"]) == 20
    for m, g in zip(suite, golden["suite"]):
        assert m.shape == (512, 512) and m.dtype == np.float32
        assert float(np.sum(m, dtype=np.float64)) == g["sum"]
        assert float(np.sum(m.astype(np.float64) ** 2)) == g["sumsq"]
        assert [float(x) for x in m[0, :4]] == g["first"]


def test_iqr_stats_matches_reference_matrix(golden):
    from paper_2405_12591_b200.analysis import iqr_stats, synth_activations

    st = iqr_stats(synth_activations(512, 512, 8, 20.0, seed=0))
    g = golden["migration"]["matrix"]
    assert (st.q1, st.q3, st.iqr, st.outlier_count, st.total_count) == (g["q1"], g["q3"], g["iqr"], g["outlier_count"],
                                                                        g["total"])
