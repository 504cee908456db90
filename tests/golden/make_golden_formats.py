"""Golden DQT1 / DQZ1 files written by the REFERENCE (formats.py), for byte-level parity.

    python tests/golden/make_golden_formats.py   ->  tests/golden/golden_formats.json

Build container only (imports /root/reference/pkg/src read-only).  Each entry holds the
input (as fp16-exact values) and the reference's file bytes (hex).
"""

from __future__ import annotations

import json
import os
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from dquant import QuantizedTensor, deco_quantize, pack
    from dquant.formats import write_mpo, write_tensor

    out = {"reference": REF}
    tmp = tempfile.mkdtemp()

    def file_hex(write, obj):
        p = os.path.join(tmp, "x")
        write(p, obj)
        with open(p, "rb") as f:
            return f.read().hex()

    t = np.random.default_rng(3).standard_normal((5, 7, 2)).astype(np.float16).astype(np.float32)
    out["float_tensor"] = {"values": t.ravel().tolist(), "shape": list(t.shape), "file": file_hex(write_tensor, t)}
    q = QuantizedTensor(shape=(3, 5), bits=4, scale=0.25, payload=pack(list(range(-7, 8)), 4))
    out["packed_tensor"] = {"codes": list(range(-7, 8)), "shape": [3, 5], "bits": 4, "scale": 0.25,
                            "file": file_hex(write_tensor, q)}
    chains = []
    for seed, (rows, cols, bits) in enumerate([(64, 48, 4), (256, 128, 2), (512, 128, 4), (1009, 128, 8)]):
        m = np.random.default_rng(40 + seed).standard_normal((rows, cols)).astype(np.float16).astype(np.float32)
        chains.append({"rows": rows, "cols": cols, "bits": bits, "seed": 40 + seed,
                       "file": file_hex(write_mpo, deco_quantize(m, bits))})
    out["chains"] = chains
    with open(os.path.join(HERE, "golden_formats.json"), "w") as f:
        json.dump(out, f)
    print("wrote golden_formats.json", [len(c["file"]) // 2 for c in chains])


if __name__ == "__main__":
    main()
