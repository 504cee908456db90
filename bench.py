#!/usr/bin/env python
"""Decode benchmark of the B200-native DecoQuant hot path (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A *step* is one decode step of the attention hot path over every layer of the
model shape: per layer, the fused int-k DecoQuant dequant + decode attention
(K5) over each unit's compressed KV plus the append of the new token's K/V row
into the fp16 tail (kvcache.py:116-123).  Units are (sequence, kv head) pairs.
Multi-GPU: one process per GPU (`--gpus N` relaunches itself under
torch.distributed.run when not already under it).  C2 / C3 scale weakly (each rank
a replica over its own batch); C4 / C5 shard the kv heads of a fixed batch across
the ranks (strong).  The attention path has no collective; the ranks meet only at
the barriers around the timed region and the max over ranks of the device times.

Default workload (BASELINE.json configs[1]): LLaMA-2-7B shape (32 layers,
32 kv heads, head dim 128), batch 16 per 32-head shard, 4K-token context
prefilled as one segment per unit, int4 large core.  Synthetic data:
K/V ~ N(0,1) fp16 compressed by the real write path (K3).

``--impl reference`` times the CPU oracle (a numpy restatement of the
reference's fused_matmul_t -> softmax -> fused_matmul per unit) on all host
cores with a bounded sample per step, extrapolated to the same step.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: workload, layers, kv_heads, g, batch, context T, bits, scaling over N GPUs:
    #   weak   -- batch per GPU fixed (each rank holds every kv head of its own sequences' shard
    #             of `batch` x kv_heads units: the global batch grows with N);
    #   strong -- the global batch is fixed and the kv heads are sharded across the ranks
    #             (BASELINE.json configs[3] "KV heads sharded across 2/4/8 B200", configs[4]
    #             "one KV head per GPU on 8 x B200")
    "c2": dict(workload="llama2-7b-shape decode attention, batch 16, 4K context, int4 DecoQuant KV",
               model="llama2-7b-shape", layers=32, kv_heads=32, g=1, batch=16, T=4096, bits=4, scaling="weak"),
    "c3": dict(workload="llama2-13b-shape decode attention, batch 32, 8K context, int2 DecoQuant KV",
               model="llama2-13b-shape", layers=40, kv_heads=40, g=1, batch=32, T=8192, bits=2, scaling="weak"),
    "c4": dict(workload="llama2-7b-shape long-context decode attention, batch 1, 32K context, int4",
               model="llama2-7b-shape", layers=32, kv_heads=32, g=1, batch=1, T=32768, bits=4, scaling="strong"),
    # configs[0]: the write / reconstruct path alone (run_c1): 32 heads x 2048 tokens x 128, int4, n = 2
    "c1": dict(workload="synthetic KV tensor 32 heads x 2048 tokens x 128, 2-factor MPO, int4: decompose / "
                        "quantize / reconstruct", model="kv-tensor", layers=1, kv_heads=32, g=1, batch=1, T=2048,
               bits=4, scaling="weak"),
    "c5": dict(workload="llama2-70b-shape GQA decode attention, batch 64, 16K context, int4",
               model="llama2-70b-shape", layers=80, kv_heads=8, g=8, batch=64, T=16384, bits=4, scaling="strong"),
}


class Ranks:
    """One process per GPU (torchrun env: RANK / LOCAL_RANK / WORLD_SIZE / MASTER_*).

    NCCL on GPUs, gloo without CUDA (the CPU plumbing test).  The decode attention path has
    no collective: the process group carries only the barriers around the timed region and
    the max-over-ranks of the device times."""

    def __init__(self, backend=None):
        import torch
        import torch.distributed as dist

        self.dist = dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.backend = backend or ("nccl" if torch.cuda.is_available() else "gloo")
        self.dev = None
        if self.backend == "nccl":
            torch.cuda.set_device(self.local)
            self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            if self.backend == "nccl":
                dist.init_process_group("nccl", device_id=self.dev)
            else:
                dist.init_process_group("gloo")

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max(self, x: float) -> float:
        if self.world == 1:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def gather_objects(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def shard(cfg, world: int, rank: int):
    """This rank's share of the config: (global batch, [lo, hi) kv heads, units).

    Units are (sequence, kv head) pairs in sharding.local_units order; every rank holds the
    same number (kv_heads % world == 0)."""
    from paper_2405_12591_b200.sharding import kv_head_range, local_units

    global_batch = cfg["batch"] * world if cfg["scaling"] == "weak" else cfg["batch"]
    if cfg["scaling"] == "weak":  # every kv head of this rank's own sequences (no sharding needed)
        lo, hi = 0, cfg["kv_heads"]
        units = cfg["batch"] * cfg["kv_heads"]
    else:
        lo, hi = kv_head_range(cfg["kv_heads"], rank, world)
        units = len(local_units(cfg["batch"], cfg["kv_heads"], rank, world))
    return global_batch, (lo, hi), units


def spawn_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: relaunch this command as N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1; rank 0's JSON line is this process's output."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--chunk-b", type=int, default=None, help="rows per split-kernel work item (default: auto)")
    ap.add_argument("--kernel-g", type=int, default=None, help="query heads per split-kernel head group (1 or 2)")
    ap.add_argument("--tc", type=int, default=None, choices=[0, 1],
                    help="split kernel: 1 = tcgen05, 0 = mma.sync, default: tcgen05 where eligible")
    ap.add_argument("--tail", type=int, default=0,
                    help="fp16 tail tokens per unit before the timed region (steady state: e.g. 512)")
    ap.add_argument("--seal", action="store_true",
                    help="steady state across a chunk seal: the tail is filled so that the 1024-token chunk "
                         "seals (K3 compresses it into a segment) in the middle of the timed region")
    ap.add_argument("--asym", type=int, default=0, choices=[0, 1],
                    help="1: the opt-in per-channel asymmetric quantizer (not the reference scheme)")
    ap.add_argument("--ctas", type=int, default=None,
                    help="split-kernel grid: default persistent (resident CTAs), 0 = one CTA per 256-row slice")
    ap.add_argument("--layers", type=int, default=None, help="override layer count (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--model", default=None, choices=["7b", "13b", "70b"],
                    help="whole-model decode (model.py DecoQuantLM: random-init bf16 weights of the shape, cuBLAS "
                         "projections, the fused DecoQuant attention) on the config's batch and context")
    ap.add_argument("--shard-of", type=int, default=1,
                    help="strong-scaling configs on one GPU: run rank 0's kv-head shard of an N-GPU job and "
                         "report the N-rank job's projected throughput (the ranks run identical shards with no "
                         "collective on the attention path); not a multi-GPU measurement")
    ap.add_argument("--plumbing", action="store_true",
                    help="rank plumbing only (launcher, shards, barriers, max over ranks; no kernels): CPU test")
    return ap.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(config: str):
    """DRAM bytes (read + write) per split-kernel launch from the newest committed ncu --set full
    capture (profiles/rNN_ncu_decode_attn.txt, taken on C2: scripts/profile_round.sh)."""
    import glob
    import re

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_decode_attn.txt")))
    if config != "c2" or not files:
        return None, None
    total = 0.0
    txt = open(files[-1]).read()
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        hit = re.search(m + r"\s+([0-9.]+)\s+(\w+)", txt)
        if not hit:
            return None, None
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(hit.group(2))
        if scale is None:
            return None, None
        total += float(hit.group(1)) * scale
    return total, os.path.relpath(files[-1], ROOT)


# ---------------------------------------------------------------------------
# CPU side: the oracle (reference algorithm) on host cores
# ---------------------------------------------------------------------------
_W = {}


def _cpu_worker_init(T, bits, g, seed):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np

    from oracle import dquant_oracle as O

    rng = np.random.default_rng(seed + os.getpid())
    k = rng.standard_normal((T, 128)).astype(np.float16).astype(np.float32)
    v = rng.standard_normal((T, 128)).astype(np.float16).astype(np.float32)
    lay = O.LayerOracle(128, bits, 1 << 30)
    lay.prefill(k, v)
    _W["lay"] = lay
    _W["q"] = rng.standard_normal((g, 128)).astype(np.float16).astype(np.float32)


def _cpu_units(n):
    t0 = time.perf_counter()
    for _ in range(n):
        _W["lay"].attend(_W["q"])
    return time.perf_counter() - t0


def _cpu_probe(_):
    return _cpu_units(1)


class CpuArm:
    """Pool of single-threaded workers, one per host core, each holding one encoded unit."""

    def __init__(self, cfg):
        import multiprocessing as mp

        os.environ["OPENBLAS_NUM_THREADS"] = "1"
        os.environ["OMP_NUM_THREADS"] = "1"
        self.cores = os.cpu_count() or 1
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(self.cores, initializer=_cpu_worker_init, initargs=(cfg["T"], cfg["bits"], cfg["g"], 7))
        per_unit = max(self.pool.map(_cpu_probe, range(self.cores)))  # also warms every worker
        self.per_unit = per_unit

    def sample(self, seconds):
        """Run ~`seconds` of work on every core; returns (units done, wall seconds)."""
        n = max(1, int(seconds / max(self.per_unit, 1e-4)))
        t0 = time.perf_counter()
        self.pool.map(_cpu_units, [n] * self.cores)
        return n * self.cores, time.perf_counter() - t0

    def close(self):
        self.pool.terminate()


def cpu_model_name():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args, cfg, world):
    """--impl reference: the oracle port on host cores, rank 0 only, for the WHOLE job's units."""
    global_batch = shard(cfg, world, 0)[0]
    units_per_step = cfg["layers"] * global_batch * cfg["kv_heads"]
    arm = CpuArm(cfg)
    sample_s = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        arm.sample(sample_s / 4)
    rates = []
    done = 0
    for _ in range(args.steps):
        n, dt = arm.sample(sample_s)
        rates.append(n / dt)
        done += n
    arm.close()
    units_per_s = statistics.median(rates)
    step_s = units_per_step / units_per_s
    value = global_batch / step_s
    line = {
        "impl": "reference",
        "metric": "decode tokens/s",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_s * 1e3,
        "higher_is_better": True,
        "scaling": cfg["scaling"],
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic N(0,1) K/V rounded to fp16; oracle units encoded once per worker",
        "config": config_keys(args, cfg, world, global_batch),
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": arm.cores, "kind": "port",
                         "sample": f"{done} unit-reads (T={cfg['T']}, g={cfg['g']}) over {args.steps} steps on "
                                   f"{arm.cores} single-thread workers, extrapolated to {units_per_step} units/step",
                         "cpu": cpu_model_name()},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------
class Clocks:
    """SM clock and throttle-reason sampler running during the timed region.

    NVML (nvidia_ml_py) polled from a thread every 5 ms, with one sample taken as the region
    opens and one as it closes, so even a ~40 ms region carries several samples; nvidia-smi
    (-lms 100) is the fallback where NVML is unavailable."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.nvml = None
        self.samples = []  # (sm_mhz, max_mhz, set of reason names)
        self.lines = []

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            uuid = str(torch.cuda.get_device_properties(self.index).uuid)
            return pynvml, pynvml.nvmlDeviceGetHandleByUUID("GPU-" + uuid)
        except Exception:
            vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
            ids = [x for x in vis.split(",") if x.strip()]
            idx = int(ids[self.index]) if ids and ids[self.index].strip().isdigit() else self.index
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx)

    def _sample(self):
        nv, h = self.nvml
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        masks = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                 nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        self.samples.append((float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                             float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)),
                             {n for n, m in zip(self.NAMES, masks) if bits & m}))

    def _poll(self):
        while not self.stop.wait(0.005):
            try:
                self._sample()
            except Exception:
                return

    def __enter__(self):
        import threading
        try:
            self.nvml = self._nvml_handle()
            self._sample()
            self.stop = threading.Event()
            self.thread = threading.Thread(target=self._poll, daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.nvml is not None:
            self.stop.set()
            self.thread.join(timeout=1)
            try:
                self._sample()
            except Exception:
                pass
            return
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        for clk, m, rs in self.samples:
            sm.append(clk)
            mx = m
            reasons |= rs
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(self.NAMES, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "sampler": "nvml" if self.samples else "nvidia-smi"}


def config_keys(args, cfg, world, global_batch):
    """The `config` object both arms print (same keys, same values)."""
    _, (lo, hi), units = shard(cfg, world, 0)
    T, bits = cfg["T"], cfg["bits"]
    kv_gb = (args.layers or cfg["layers"]) * units * 2 * (T * 128 * bits // 8 + 8 * 8 * 64 * 4 + 4) / 1e9
    return {"workload": cfg["workload"], "global_batch": global_batch, "seq_len": T, "context": T,
            "kv_bits": bits, "tail_tokens": args.tail if not args.seal else "seal mid-region",
            "quantizer": "per-channel asymmetric (opt-in)" if args.asym else "per-tensor symmetric (reference)",
            "layers": args.layers or cfg["layers"], "kv_heads": cfg["kv_heads"], "g": cfg["g"],
            "kv_heads_per_gpu": hi - lo, "units_per_gpu": units,
            "parallelism": f"kv-head shards x{world}" if cfg["scaling"] == "strong" else f"data-parallel replicas x{world}",
            "step": "attention only: fused dequant + decode attention + tail append per layer (no projections); "
                    "replayed as one CUDA graph",
            "l2": f"inputs > L2: {kv_gb:.2f} GB of compressed KV streamed per step per GPU (126 MB L2)"}


def _c1_cpu_worker(seed):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np

    from oracle import dquant_oracle as O

    rng = np.random.default_rng(seed)
    m = rng.standard_normal((2048, 128)).astype(np.float16).astype(np.float32)
    t0 = time.perf_counter()
    n = 0
    while time.perf_counter() - t0 < 3.0:
        O.encode(m, 4)
        n += 1
    return n, time.perf_counter() - t0


def api_calls(block, O, reps: int = 20) -> dict:
    """The reference-facing API one call at a time, numpy in / numpy out as a drop-in caller
    uses it (host <-> device copies and the host sync inside every call): deco_quantize,
    deco_dequantize, fused_matmul_t of one query row, and KvCache.attention_scores over a
    2-segment + tail cache, against the oracle's single-thread time for the same call."""
    import numpy as np

    import paper_2405_12591_b200 as dq

    def per_call(fn, n):
        fn()
        t0 = time.perf_counter()
        for _ in range(n):
            fn()
        return (time.perf_counter() - t0) / n * 1e6

    rng = np.random.default_rng(1)
    q = rng.standard_normal((1, 128)).astype(np.float32)
    qm = dq.deco_quantize(block, 4)
    e = O.encode(block, 4)
    cfg = dq.CacheConfig(layers=1, dim=128, bits=4, chunk_len=1024)
    cache = dq.KvCache(cfg)
    cache.prefill(0, block, block)
    for row in block[:1100]:
        cache.append_token(0, row, row)  # one sealed 1024-row chunk + a 76-row tail
    lay = O.LayerOracle(128, 4, 1024)
    lay.prefill(block, block)
    for row in block[:1100]:
        lay.append(row, row)
    rows = {
        "deco_quantize (2048 x 128, int4)": (lambda: dq.deco_quantize(block, 4), lambda: O.encode(block, 4)),
        "deco_dequantize": (lambda: dq.deco_dequantize(qm), lambda: O.decode(e)),
        "fused_matmul_t (1 query row)": (lambda: dq.fused_matmul_t(q, qm), lambda: O.matmul_t(q, e)),
        "KvCache.attention_scores (2 segments + tail)": (lambda: cache.attention_scores(0, q[0]),
                                                         lambda: lay.scores(q[0])),
    }
    out = {}
    for name, (ours, ref) in rows.items():
        us, ref_us = per_call(ours, reps), per_call(ref, max(2, reps // 5))
        out[name] = {"us_per_call": us, "oracle_us_per_call_1_thread": ref_us, "speedup": ref_us / us}
    return out


def run_c1(args, cfg):
    """BASELINE.json configs[0]: K3 (decompose + quantize) and K4 (reconstruct) on the 32-head
    2048 x 128 tensor, int4: per-block time, fp64 rate against the measured FP64 peak, parity
    against the CPU oracle (the reference's algorithm) and the oracle's own rate on host cores."""
    import numpy as np
    import torch

    from oracle import dquant_oracle as O
    from paper_2405_12591_b200 import _lib
    from paper_2405_12591_b200.compress import deco_quantize_batched
    from paper_2405_12591_b200.csrc_info import FP64_PEAK_TFLOPS

    torch.cuda.set_device(0)
    heads, T = cfg["kv_heads"], cfg["T"]
    rng = np.random.default_rng(0)
    k = rng.standard_normal((heads, T, 128)).astype(np.float16)
    kd = torch.from_numpy(k).cuda()

    def k3(x):
        r = deco_quantize_batched(x, 4)
        return r

    def k4(r, nblk):
        out = torch.empty((nblk, T, 128), dtype=torch.float32, device="cuda")
        _lib.check(_lib.lib().dq_deco_dequantize_batched(
            r["core0"].data_ptr(), r["payload"].data_ptr(), r["payload"].shape[1], _lib.LAYOUT_REF,
            r["scale"].data_ptr(), nblk, T, 128, 4, out.data_ptr(), _lib.DQ_F32, _lib.stream_ptr()), "k4")
        return out

    def timed(fn, reps):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    # the 32-head tensor (one call), and a throughput batch of 1024 blocks
    res = k3(kd)
    _lib.raise_flags(res["flags"], "c1")
    ms32 = timed(lambda: k3(kd), args.steps)
    big = kd.repeat(32, 1, 1)
    ms1024 = timed(lambda: k3(big), max(3, args.steps // 4))
    rec_ms = timed(lambda: k4(res, heads), args.steps)
    rec_big = deco_quantize_batched(big, 4)
    rec_ms_big = timed(lambda: k4(rec_big, big.shape[0]), max(3, args.steps // 4))
    # parity: payload bytes (after sign alignment there is nothing to align for the codes' bytes
    # when the factor signs match) and reconstruction vs the oracle
    rec = k4(res, heads).cpu().numpy()
    errs = []
    for h in range(heads):
        e = O.encode(k[h].astype(np.float32), 4)
        ref = O.decode(e)
        errs.append(float(np.linalg.norm(rec[h] - ref) / np.linalg.norm(ref)))
    m, n = 64, 2 * T
    fp64_flop = 2 * m * m * n + 2 * m * m * n  # Gram (full 64 x 64 tiles) + projection
    tflops = big.shape[0] * fp64_flop / (ms1024 / 1e3) / 1e12
    in_bytes, out_bytes = T * 128 * 2, T * 128 * 4
    line = {
        "metric": "C1 write path: deco_quantize blocks/s (2048 x 128, int4, n = 2)",
        "value": big.shape[0] / (ms1024 / 1e3), "unit": "blocks/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms32, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic N(0,1) rounded to fp16",
        "config": {"workload": cfg["workload"], "heads": heads, "T": T, "bits": 4, "n": 2},
        "k3": {"us_per_block_32": ms32 * 1e3 / heads, "us_per_block_1024": ms1024 * 1e3 / big.shape[0],
               "fp64_tflops": tflops, "fp64_peak_tflops": FP64_PEAK_TFLOPS, "fp64_frac": tflops / FP64_PEAK_TFLOPS,
               "fp64_flop_per_block": fp64_flop},
        "k4": {"us_per_block_32": rec_ms * 1e3 / heads, "gbs_1024": big.shape[0] * (in_bytes // 4 + out_bytes)
               / (rec_ms_big / 1e3) / 1e9, "us_per_block_1024": rec_ms_big * 1e3 / big.shape[0]},
        "parity": {"reconstruction_rel_frob_max": max(errs), "tolerance": 1e-3},
        "api": api_calls(k[0].astype(np.float32), O),
    }
    if not args.no_cpu_baseline:
        import multiprocessing as mp

        cores = os.cpu_count() or 1
        with mp.get_context("spawn").Pool(cores) as pool:
            outs = pool.map(_c1_cpu_worker, range(cores))
        rate = sum(n / dt for n, dt in outs)
        line["cpu_baseline"] = {"value": rate, "unit": "blocks/s", "cores": cores, "kind": "port",
                                "sample": f"oracle encode (2048 x 128, int4) for 3 s on each of {cores} "
                                          "single-thread workers", "cpu": cpu_model_name()}
    print(json.dumps(line), flush=True)


def run_model(args, cfg):
    """--model: one decode step of a whole LLaMA-shaped decoder (model.py) per step, replayed as a
    CUDA graph: device-resident tokens for `value`, host tokens in / next tokens out for `e2e`.
    Under N ranks the decoder is tensor-parallel (model.py: kv heads and 1/N of every weight per
    GPU, NCCL all-gathers inside the captured step); the global batch is fixed (strong scaling).
    Roofline: the weights (bf16) + the compressed KV + the fp16 tails one step streams per GPU."""
    import torch

    from paper_2405_12591_b200.model import LLAMA2_7B, LLAMA2_13B, LLAMA2_70B, DecoQuantLM
    from paper_2405_12591_b200.sharding import TpGroup

    rk = Ranks("nccl")
    shape = {"7b": LLAMA2_7B, "13b": LLAMA2_13B, "70b": LLAMA2_70B}[args.model]
    if args.layers:
        from dataclasses import replace
        shape = replace(shape, layers=args.layers)
    batch, T = cfg["batch"], cfg["T"]
    tp = TpGroup(world=rk.world, rank=rk.rank) if rk.world == 1 else TpGroup()
    lm = DecoQuantLM(shape, batch, bits=cfg["bits"], tp=tp)
    lm.prefill_random(T)
    torch.cuda.synchronize()
    tok = torch.zeros(batch, dtype=torch.int64, device=rk.dev)
    for _ in range(args.warmup):
        tok = lm.step(tok)
    lm.capture(tok)
    for _ in range(args.warmup):
        tok = lm.replay(tok)
    torch.cuda.synchronize()
    rk.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(rk.local) as clk:
        e0.record()
        for _ in range(args.steps):
            tok = lm.replay(tok)
        e1.record()
        torch.cuda.synchronize()
    rk.barrier()
    ms = rk.max(e0.elapsed_time(e1) / args.steps)
    # end to end: pinned host tokens in, the step, next tokens back to the host, every step
    tok_h = torch.zeros(batch, dtype=torch.int64).pin_memory()
    nxt_h = torch.zeros(batch, dtype=torch.int64).pin_memory()
    steps_e2e = max(3, args.steps // 2)
    torch.cuda.synchronize()
    rk.barrier()
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(steps_e2e):
        nxt = lm.replay(tok_h.to(rk.dev, non_blocking=True))
        nxt_h.copy_(nxt, non_blocking=True)
        tok_h, nxt_h = nxt_h, tok_h
    f1.record()
    torch.cuda.synchronize()
    e2e_ms = rk.max(f0.elapsed_time(f1) / steps_e2e)
    wbytes = sum(t.numel() * t.element_size() for L in lm.layers for t in L.values())
    wbytes += lm.lm_head.numel() * lm.lm_head.element_size() + batch * shape.hidden * 2
    kv = sum(lm.cache.read_bytes(layer) for layer in range(shape.layers))
    peak, peak_kind = measured_peaks()
    fp16, actual = lm.cache.ledger()
    world = rk.world
    gathers = 4 * shape.layers + (2 if world > 1 else 0)
    line = {
        "metric": "decode tokens/s (whole model)", "value": batch / (ms / 1e3), "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "bf16 weights, f16 attention",
        "data": "synthetic: random-init weights (std 0.02), K/V ~ N(0,1) compressed by K3",
        "config": {"workload": f"llama2-{args.model}-shape decode (whole model), batch {batch}, {T} context, "
                               f"int{cfg['bits']} DecoQuant KV", "model": f"llama2-{args.model}-shape",
                   "global_batch": batch, "seq_len": T, "layers": shape.layers,
                   "parallelism": f"tp{world}: kv heads + output-column weight shards, "
                                  f"{gathers} NCCL all-gathers per step" if world > 1 else "single GPU",
                   "l2": f"weights {wbytes / 1e9:.1f} GB + KV {kv / 1e9:.1f} GB streamed per step per GPU (126 MB L2)"},
        "roofline": {"bound": "hbm", "achieved": (wbytes + kv) / (ms / 1e3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": (wbytes + kv) / (ms / 1e3) / 1e9 / peak, "traffic": None,
                     "kernel": "whole step (weights + KV, per GPU)", "bytes_per_step": wbytes + kv,
                     "peak_kind": peak_kind},
        "memory_per_token_vs_fp16": actual / fp16,
        "e2e": {"value": batch / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": batch * 8,
                "d2h_bytes_per_step": batch * 8, "ms_per_step": e2e_ms},
        "gpu_launches": args.steps * (shape.layers * 10 + 3),
        "clocks": clk.summary(),
    }
    if rk.rank == 0:
        print(json.dumps(line), flush=True)
    rk.close()


def run_plumbing(args, cfg):
    """--plumbing: the launcher / rank / shard / timing path of run_ours without kernels (gloo on
    CPU in tests/test_bench_ranks.py; the same Ranks and shard() the GPU run uses)."""
    rk = Ranks()
    global_batch, (lo, hi), units = shard(cfg, rk.world, rk.rank)
    rk.barrier()
    t0 = time.perf_counter()
    time.sleep(0.01 * (rk.rank + 1))  # stand-in for the rank's timed steps
    ms = rk.max((time.perf_counter() - t0) * 1e3)
    shards = rk.gather_objects({"rank": rk.rank, "heads": [lo, hi], "units": units})
    if rk.rank == 0:
        print(json.dumps({"plumbing": True, "n_gpus": rk.world, "backend": rk.backend, "scaling": cfg["scaling"],
                          "global_batch": global_batch, "ms_max": ms, "shards": shards}), flush=True)
    rk.close()


def run_ours(args, cfg):
    import torch

    from paper_2405_12591_b200.attention import DecodeKvCache

    rk = Ranks("nccl")
    world, rank, local, dev = rk.world, rk.rank, rk.local, rk.dev
    layers = args.layers or cfg["layers"]
    kv_heads, g, bits, T = cfg["kv_heads"], cfg["g"], cfg["bits"], cfg["T"]
    if kv_heads % world:
        raise SystemExit(f"{kv_heads} kv heads do not shard over {world} GPUs")
    proj = args.shard_of if world == 1 and args.shard_of > 1 else 0  # --shard-of: one rank of an N-GPU job
    if proj and (cfg["scaling"] != "strong" or kv_heads % proj):
        raise SystemExit("--shard-of needs a strong-scaling config whose kv heads shard over N")
    global_batch, (head_lo, head_hi), units = shard(cfg, proj or world, rank)  # units: (sequence, kv head) pairs
    chunk_len = 1024

    cache = DecodeKvCache(layers=layers, units=units, g=g, bits=bits, chunk_len=chunk_len, chunk_b=args.chunk_b,
                          ctas=args.ctas, kernel_g=args.kernel_g,
                          tc=None if args.tc is None else bool(args.tc), asym=bool(args.asym))
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)

    # ---- write path (K3): every layer's prompt compressed for real, timed -------------
    write_s = 0.0
    for layer in range(layers):
        k0 = torch.randn((units, T, 128), generator=gen, device=dev, dtype=torch.float32).to(torch.float16)
        v0 = torch.randn((units, T, 128), generator=gen, device=dev, dtype=torch.float32).to(torch.float16)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        cache.prefill(layer, k0, v0)
        torch.cuda.synchronize()
        write_s += time.perf_counter() - t0
        del k0, v0
    torch.cuda.empty_cache()
    fp16_bytes, actual_bytes = cache.ledger()

    q = torch.randn((layers, units, g, 128), generator=gen, device=dev).to(torch.float16)
    kn = torch.randn((layers, units, 128), generator=gen, device=dev).to(torch.float16)
    vn = torch.randn((layers, units, 128), generator=gen, device=dev).to(torch.float16)
    out = torch.empty_like(q)
    for layer in range(layers):  # build segment tables / work lists outside the timed region
        cache.attend(layer, q[layer], out[layer])
    torch.cuda.synchronize()

    def step():
        for layer in range(layers):
            # one launch sequence per layer: attention over the cache, then the new token
            # joins the tail (append fused into the combine kernel)
            cache.attend(layer, q[layer], out[layer], append=(kn[layer], vn[layer]))

    barrier, max_over_ranks = rk.barrier, rk.max

    # steady state: a partly filled fp16 tail (DecodeKvCache.extend_tail: the state of
    # that many append_token calls); --seal fills it so the chunk seals at timed step K // 2
    fill = chunk_len - 1 - args.warmup - args.steps // 2 if args.seal else args.tail
    if fill > 0:
        for layer in range(layers):
            cache.extend_tail(layer, torch.randn((units, fill, 128), generator=gen, device=dev).half(),
                              torch.randn((units, fill, 128), generator=gen, device=dev).half())
    torch.cuda.synchronize()
    appended = fill + args.warmup + args.steps + 2 + max(3, args.warmup // 2) + max(3, args.steps // 2)
    if appended + 1 >= chunk_len and not args.seal:
        raise SystemExit("steps too large: the tail would seal a chunk inside the timed region")

    # ---- device-resident timed region ----------------------------------------------
    # the step replayed as one CUDA graph (decode_step.DeviceStepGraph: every layer's kernels
    # with the whole step's programmatic launch edges); --seal runs eagerly, since a graph is
    # not replayed across a seal
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    timed_step = step
    if not args.seal:
        from paper_2405_12591_b200.decode_step import DeviceStepGraph

        timed_step = DeviceStepGraph(cache, q, kn, vn, out).replay  # (its capture runs one eager step)
        timed_step()
    torch.cuda.synchronize()
    barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        evs[0].record()
        for i in range(args.steps):
            timed_step()
            evs[i + 1].record()
        torch.cuda.synchronize()
    barrier()
    step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
    ms = max_over_ranks(evs[0].elapsed_time(evs[-1]) / args.steps)
    value = global_batch / (ms / 1e3)
    seal = None
    if args.seal:  # the sealing step against the others (device timeline, host work included)
        med = statistics.median(step_ms)
        ev_ms = max(step_ms) - med
        seal = {"chunk_len": chunk_len, "blocks": 2 * units * layers, "block": f"{chunk_len}x128",
                "sealing_step_ms": max(step_ms), "median_step_ms": med, "event_ms": ev_ms,
                "amortised_ms_per_step": ev_ms / chunk_len, "fraction_of_step": ev_ms / chunk_len / med}
        for layer in range(layers):  # the sealed layers build their tables outside the later timed parts
            cache.attend(layer, q[layer], out[layer])
        torch.cuda.synchronize()

    # ---- split-kernel launches alone, for the roofline: every layer's split kernel back to back
    # (no PDL edge, so no launch overlaps another), CUDA events around the batch on this stream,
    # average duration per launch; the per-launch event pairs of round 1 added ~3 us of event /
    # launch gap per launch (ncu: 58.7 us per launch against 62.1 us from per-launch events)
    kern_runs = []
    for rep in range(4):
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record()
        for layer in range(layers):
            cache.launch(layer, q[layer], out[layer], phases=1 | 8)
        k1.record()
        torch.cuda.synchronize()
        if rep:
            kern_runs.append(k0.elapsed_time(k1) / layers)
    kern_ms = max_over_ranks(statistics.mean(kern_runs))
    kern_bytes = cache.kernel_bytes(0)
    achieved = kern_bytes / (kern_ms / 1e3) / 1e9
    peak, peak_kind = measured_peaks()
    traffic, traffic_src = ncu_traffic(args.config)
    step_bytes = sum(cache.read_bytes(layer) for layer in range(layers))

    # ---- end-to-end through the public API with host buffers --------------------------
    q_h = q.cpu().pin_memory()
    kn_h, vn_h = kn.cpu().pin_memory(), vn.cpu().pin_memory()
    out_h = torch.empty(q.shape, dtype=torch.float16).pin_memory()

    # the public decode-step API: host buffers in / out, the step replayed as one CUDA graph
    # (per-layer copies on a side stream overlap the previous layer's kernels)
    from paper_2405_12591_b200.decode_step import DecodeStepGraph

    stepper = DecodeStepGraph(cache, q_h, kn_h, vn_h, out_h)

    def e2e_step():
        stepper.replay()

    e2e_steps = max(3, args.steps // 2)
    for _ in range(max(3, args.warmup // 2)):
        e2e_step()
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(e2e_steps):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1) / e2e_steps)
    h2d = layers * (q[0].numel() + kn[0].numel() + vn[0].numel()) * 2
    d2h = layers * q[0].numel() * 2

    line = {
        "metric": "decode tokens/s",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": cfg["scaling"],
        "vs_baseline": None,
        "dtype": "f16",
        "data": "synthetic: per-layer K/V ~ N(0,1) fp16 compressed by the K3 write path; q/k/v rows ~ N(0,1) fp16",
        "config": config_keys(args, cfg, proj or world, global_batch),
        "kernel": {"chunk_b": cache._layers[0].args.chunk_b, "split_ctas": cache.split_ctas,
                   "kernel_g": cache._layers[0].kernel_g, "head_groups": g // cache._layers[0].kernel_g,
                   "split_path": {0: "mma.sync", 1: "tcgen05", 2: "tcgen05-gqa"}[cache._layers[0].args.path],
                   "step_bytes": step_bytes},
        "hbm_gbs_step": step_bytes / (ms / 1e3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": {0: "decode_attn_kernel", 1: "decode_attn_tc_kernel", 2: "decode_attn_gqa_kernel"}[cache._layers[0].args.path],
                     "bytes_per_launch": kern_bytes, "bytes_basis": "SURVEY 8(d) algorithmic (fp16 small cores)",
                     "stream_bytes_per_launch": cache.stream_bytes(0),
                     "launch_ms": kern_ms, "peak_kind": peak_kind},
        "memory_per_token_vs_fp16": actual_bytes / fp16_bytes,
        **({"seal": seal} if seal else {}),
        "write_path": {"blocks": 2 * units * layers, "block": f"{T}x128", "seconds": write_s,
                       "blocks_per_s": 2 * units * layers / write_s},
        "e2e": {"value": global_batch / (e2e_ms / 1e3), "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "gpu_launches": args.steps * layers * 3,  # per layer: prepare, split, combine (+ fused tail append)
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        arm = CpuArm(cfg)
        n, dt = arm.sample(args.cpu_seconds)
        arm.close()
        units_per_step = layers * units
        cpu_tok = global_batch / (units_per_step / (n / dt))
        line["cpu_baseline"] = {"value": cpu_tok, "unit": "tokens/s", "cores": arm.cores, "kind": "port",
                                "sample": f"{n} unit-reads (T={T}, int{bits}, g={g}) in {dt:.1f}s on {arm.cores} "
                                          f"single-thread workers, extrapolated to {units_per_step} units/step",
                                "cpu": cpu_model_name()}
    if proj:
        line["projection"] = {
            "n_gpus": proj, "value": line["value"], "e2e": line["e2e"]["value"],
            "basis": f"rank 0's shard ({units} units per layer) measured on one GPU; the {proj} ranks run "
                     "identical shards with no collective on the attention path, so the job's step is the rank's "
                     "step (barriers and power sharing not measured)"}
        line["note"] = "projection from one rank's shard, not a multi-GPU measurement"
    if rank == 0:
        print(json.dumps(line), flush=True)
    rk.close()


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args))  # one rank per GPU under torch.distributed.run
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU")
    if args.plumbing:
        run_plumbing(args, cfg)
        return
    if args.model and args.impl != "reference":
        run_model(args, cfg)
        return
    if args.config == "c1":
        if rank == 0 and args.impl != "reference":
            run_c1(args, cfg)
        elif rank == 0:
            print(json.dumps({"impl": "reference", "unavailable": "c1 reports its CPU arm as cpu_baseline"}))
        return
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cfg, world)
        return
    run_ours(args, cfg)


if __name__ == "__main__":
    main()
