"""DQT1 float tensors and malformed-file handling of the DQT1 / DQZ1 reader (CPU; the packed
cases need the device codec and live in test_gpu_formats.py)."""

import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def golden():
    with open(os.path.join(HERE, "golden", "golden_formats.json")) as f:
        return json.load(f)


def test_float_tensor_bytes_match_reference(golden, tmp_path):
    from paper_2405_12591_b200.formats import read_tensor, tensor_bytes, write_tensor

    g = golden["float_tensor"]
    t = np.array(g["values"], np.float32).reshape(g["shape"])
    assert tensor_bytes(t).hex() == g["file"]
    p = tmp_path / "t.dqt"
    write_tensor(p, t)
    back = read_tensor(p)
    assert back.dtype == np.float32 and np.array_equal(back, t)


def test_malformed_files(tmp_path, golden):
    from paper_2405_12591_b200.errors import MalformedFile
    from paper_2405_12591_b200.formats import parse_mpo, read_tensor

    good = bytes.fromhex(golden["float_tensor"]["file"])
    cases = {
        "magic": b"DQT0" + good[4:],
        "truncated": good[:-3],
        "trailing": good + b"\0",
        "kind": good[:4] + b"\x07" + good[5:],
    }
    for name, data in cases.items():
        p = tmp_path / f"{name}.dqt"
        p.write_bytes(data)
        with pytest.raises(MalformedFile):
            read_tensor(p)
    chain = bytes.fromhex(golden["chains"][0]["file"])
    for data in (b"DQZ0" + chain[4:], chain[:4] + b"\x02" + chain[5:], chain[:5] + b"\x01" + chain[6:], chain[:-1]):
        with pytest.raises(MalformedFile):
            parse_mpo(data)
