"""bench.py's multi-GPU launcher and rank plumbing on CPU (gloo, world size 2).

`bench.py --gpus N` outside torchrun relaunches itself as N ranks under
torch.distributed.run (bench.spawn_ranks); every rank builds the same Ranks /
shard() objects the GPU run uses.  --plumbing stops before the kernels: each rank
times a stand-in step, rank 0 reports the max over ranks and the shards.
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*argv):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], capture_output=True, text=True,
                         timeout=300, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [ln for ln in res.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, res.stdout  # exactly one JSON line, from rank 0
    return json.loads(lines[0])


@pytest.mark.parametrize("config,scaling", [("c4", "strong"), ("c5", "strong"), ("c2", "weak")])
def test_launcher_world2(config, scaling):
    d = _run("--gpus", "2", "--plumbing", "--config", config)
    assert d["n_gpus"] == 2 and d["backend"] == "gloo" and d["scaling"] == scaling
    assert d["ms_max"] >= 20.0  # rank 1 sleeps 20 ms: the max over ranks, not rank 0's own time
    shards = sorted(d["shards"], key=lambda x: x["rank"])
    assert [s["rank"] for s in shards] == [0, 1]
    import bench

    cfg = bench.CONFIGS[config]
    if scaling == "strong":  # kv heads split, every head exactly once, batch fixed
        assert shards[0]["heads"][0] == 0 and shards[0]["heads"][1] == shards[1]["heads"][0]
        assert shards[1]["heads"][1] == cfg["kv_heads"]
        assert d["global_batch"] == cfg["batch"]
        assert sum(s["units"] for s in shards) == cfg["batch"] * cfg["kv_heads"]
    else:  # weak: each rank holds its own sequences' full head set
        assert d["global_batch"] == 2 * cfg["batch"]
        assert all(s["units"] == cfg["batch"] * cfg["kv_heads"] for s in shards)


def test_world_mismatch_rejected():
    env = {k: v for k, v in os.environ.items()}
    env.update(WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plumbing"],
                         capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert res.returncode != 0 and "WORLD_SIZE" in res.stderr
