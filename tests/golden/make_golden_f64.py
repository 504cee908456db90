"""Golden vectors for quantize_rtn on float64 input, from the REFERENCE ``dquant``.

    python tests/golden/make_golden_f64.py     # build container only (/root/reference)

The reference multiplies the original values in float64 (quantize.py:144), so a
float64 input near a rounding tie (2.5 - 1e-12) or above the fp32 range must not be
rounded to fp32 first.  Writes tests/golden/golden_f64.npz.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    sys.path.insert(0, REF)
    from dquant import quantize

    rng = np.random.default_rng(64)
    cases = {
        "tie": np.array([7.0, 2.5 - 1e-12, -2.5 + 1e-12, 0.5 + 1e-13, 3.5000000000001, -7.0]),
        "huge": np.array([1e300, -3e299, 2.4e299, 5e-300]),
        "tiny": np.array([1e-310, -2e-310, 0.0]),
        "rand": rng.standard_normal(3001) * rng.choice([1e-3, 1.0, 1e5], 3001),
    }
    # values k * amax / qmax +- 1 ulp: the ties of every code level
    for bits in (2, 4, 8):
        q = (1 << (bits - 1)) - 1
        lv = np.arange(-q, q) + 0.5  # amax = q: the code levels are the integers, ties at k + 1/2
        cases[f"ties{bits}"] = np.concatenate([[float(q)], lv, np.nextafter(lv, 0), np.nextafter(lv, 10 * lv),
                                               lv - 1e-12 * np.sign(lv)])
    out = {}
    for name, t in cases.items():
        t = t.astype(np.float64)
        out[f"{name}_t"] = t
        for bits in (2, 4, 8):
            r = quantize.quantize_rtn(t, bits)
            out[f"{name}_{bits}_scale"] = np.float32(r.scale)
            out[f"{name}_{bits}_payload"] = np.frombuffer(r.payload, np.uint8)
    np.savez_compressed(os.path.join(HERE, "golden_f64.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
