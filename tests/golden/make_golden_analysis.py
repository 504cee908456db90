"""Golden quantisation-error statistics from the REFERENCE ``dquant`` sweeps.

    python tests/golden/make_golden_analysis.py

Runs the reference's own ``analysis`` module (analysis.py:147-293) on its default outlier
suite and writes ``tests/golden/golden_analysis.json``:

- ``suite``: per-seed checksums of ``default_suite()`` (20 seeds, 512 x 512, 8 outlier
  columns x 20), so a restated generator can be checked to reproduce the same matrices;
- ``strategy``: ``strategy_sweep(suite)`` records (matrix RTN / DecoQuant large core only /
  both cores, bits 2, 4, 8) and their medians -- the paper's error table;
- ``length``: ``length_sweep(suite)`` (chain length n = 2, 3, 4, large cores quantized, 4 bits);
- ``decomposition``: ``decomposition_comparison(suite)`` (chain vs SVD vs QR, 4 bits);
- ``migration``: ``migration_report`` IQR statistics of seed 0 (matrix, large, small core).

Like ``make_golden.py`` it only runs in the build container, where ``/root/reference``
exists; the JSON travels with the repo.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _records(recs):
    return [
        {"method": r.method, "bits": r.bits, "n": r.n, "seed": r.seed, "frobenius_error": r.frobenius_error,
         "relative_error": r.relative_error, "param_overhead": r.param_overhead}
        for r in recs
    ]


def _stats(st):
    return {"q1": st.q1, "q3": st.q3, "iqr": st.iqr, "outlier_count": st.outlier_count, "total": st.total_count}


def main():
    sys.path.insert(0, REF)
    from dquant import analysis

    suite = analysis.default_suite()
    out = {
        "reference": REF,
        "numpy": np.__version__,
        "suite": [{"seed": s, "sum": float(np.sum(m, dtype=np.float64)), "sumsq": float(np.sum(m.astype(np.float64) ** 2)),
                   "first": [float(x) for x in m[0, :4]]} for s, m in enumerate(suite)],
    }
    strat = analysis.strategy_sweep(suite)
    out["strategy"] = _records(strat)
    out["strategy_median"] = {f"{k[0]}/{k[1]}": v for k, v in analysis.median_by(strat).items()}
    length = analysis.length_sweep(suite)
    out["length"] = _records(length)
    out["length_median"] = {f"{k[0]}/{k[1]}": v for k, v in analysis.median_by(length, key=lambda r: (r.method, r.n)).items()}
    dec = analysis.decomposition_comparison(suite)
    out["decomposition"] = _records(dec)
    out["decomposition_median"] = {f"{k[0]}/{k[1]}": v for k, v in analysis.median_by(dec).items()}
    mat, large, small = analysis.migration_report(suite[0])
    out["migration"] = {"matrix": _stats(mat), "large": _stats(large), "small": _stats(small)}
    with open(os.path.join(HERE, "golden_analysis.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote golden_analysis.json:", {k: v for k, v in out["strategy_median"].items()})


if __name__ == "__main__":
    main()
