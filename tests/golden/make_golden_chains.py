"""Golden vectors for chains longer than 2 from the REFERENCE ``dquant``.

    python tests/golden/make_golden_chains.py

For a few matrices and n = 3, 4 runs the reference's ``plan_shapes``, ``decompose``,
``reconstruct``, ``deco_quantize`` (4 and 2 bits), ``deco_dequantize``, ``fused_matmul``,
``fused_matmul_t`` and ``compression_report`` (mpo.py:73-198, compress.py:85-248) and writes
``tests/golden/golden_chains.npz`` + ``golden_chains.json``.  Like the other generators it
only runs in the build container, where ``/root/reference`` exists.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from dquant import analysis, compress, mpo

    rng = np.random.default_rng(7)
    mats = {
        "synth256": analysis.synth_activations(256, 256, 8, 20.0, seed=3),
        "k1024": rng.standard_normal((1024, 128)).astype(np.float16).astype(np.float32),
        "r96x80": rng.standard_normal((96, 80)).astype(np.float32),
    }
    arrays, meta = {}, {"reference": REF, "numpy": np.__version__, "cases": {}}
    for name, m in mats.items():
        arrays[f"{name}_m"] = m
        for n in (3, 4):
            plan = mpo.plan_shapes(m.shape[0], m.shape[1], n)
            chain = mpo.decompose(m, plan)
            key = f"{name}_n{n}"
            arrays[f"{key}_rec"] = mpo.reconstruct(chain)
            case = {"i": list(plan.i_factors), "j": list(plan.j_factors), "bonds": list(chain.bond_dims), "bits": {}}
            x = rng.standard_normal((3, m.shape[0])).astype(np.float32)
            xt = rng.standard_normal((2, m.shape[1])).astype(np.float32)
            arrays[f"{key}_x"], arrays[f"{key}_xt"] = x, xt
            for bits in (4, 2):
                q = compress.deco_quantize(m, bits, n)
                kb = f"{key}_b{bits}"
                arrays[f"{kb}_deq"] = compress.deco_dequantize(q)
                arrays[f"{kb}_mm"] = compress.fused_matmul(x, q)
                arrays[f"{kb}_mmt"] = compress.fused_matmul_t(xt, q)
                rep = compress.compression_report(q)
                case["bits"][str(bits)] = {"ratio": rep.ratio, "bytes_compressed": rep.bytes_compressed,
                                           "scales": [t.scale for t in q.quantized_locals]}
            meta["cases"][key] = case
    np.savez_compressed(os.path.join(HERE, "golden_chains.npz"), **arrays)
    with open(os.path.join(HERE, "golden_chains.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print("wrote golden_chains:", {k: (v["i"], v["j"], v["bonds"]) for k, v in meta["cases"].items()})


if __name__ == "__main__":
    main()
