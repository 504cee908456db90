"""The oracle's chain restatement (n = 3, 4) against the reference's own outputs
(tests/golden/golden_chains.*, made by make_golden_chains.py).  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import dquant_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def gold():
    g = np.load(os.path.join(HERE, "golden", "golden_chains.npz"))
    with open(os.path.join(HERE, "golden", "golden_chains.json")) as f:
        return g, json.load(f)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30))


def test_chain_oracle_matches_reference(gold):
    g, meta = gold
    assert len(meta["cases"]) == 6
    for key, case in meta["cases"].items():
        name, n = key.rsplit("_n", 1)[0], int(key.rsplit("_n", 1)[1])
        m = g[f"{name}_m"]
        i_f, j_f = O.plan(*m.shape, n)
        assert list(i_f) == case["i"] and list(j_f) == case["j"] and list(O.bonds(i_f, j_f)) == case["bonds"]
        assert rel(g[f"{key}_rec"], O.contract(O.tt_split(m, i_f, j_f))) < 1e-6, key
        for bits in (4, 2):
            _, quant, deq = O.deco_chain(m, bits, n)
            kb = f"{key}_b{bits}"
            assert [float(s) for s, _ in quant] == case["bits"][str(bits)]["scales"], kb
            assert rel(g[f"{kb}_deq"], O.contract(deq)) < 1e-6, kb
            assert rel(g[f"{kb}_mm"], O.chain_matmul(g[f"{key}_x"], deq)) < 1e-6, kb
            assert rel(g[f"{kb}_mmt"], O.chain_matmul_t(g[f"{key}_xt"], deq)) < 1e-6, kb
