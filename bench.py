#!/usr/bin/env python
"""Decode benchmark of the B200-native DecoQuant hot path (driver contract: one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A *step* is one decode step of the attention hot path over every layer of the
model shape: per layer, the fused int-k DecoQuant dequant + decode attention
(K5) over each unit's compressed KV plus the append of the new token's K/V row
into the fp16 tail (kvcache.py:116-123).  Units are (sequence, kv head) pairs;
the KV cache is sharded by kv head across ranks (no collective on this path),
and the global batch grows with N so per-GPU work is fixed ("weak").

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
    # name: (workload, layers, kv_heads, g, batch per 32-head-equivalent shard, context, bits)
    "c2": dict(workload="llama2-7b-shape decode, batch 16, 4K context, int4 DecoQuant KV", model="llama2-7b-shape",
               layers=32, kv_heads=32, g=1, batch=16, T=4096, bits=4),
    "c3": dict(workload="llama2-13b-shape decode, batch 32, 8K context, int2 DecoQuant KV", model="llama2-13b-shape",
               layers=40, kv_heads=40, g=1, batch=32, T=8192, bits=2),
    "c4": dict(workload="llama2-7b-shape long-context decode, batch 1, 32K context, int4", model="llama2-7b-shape",
               layers=32, kv_heads=32, g=1, batch=1, T=32768, bits=4),
    "c5": dict(workload="llama2-70b-shape GQA decode, batch 64, 16K context, int4", model="llama2-70b-shape",
               layers=80, kv_heads=8, g=8, batch=64, T=16384, bits=4),
}


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
    ap.add_argument("--asym", type=int, default=0, choices=[0, 1],
                    help="1: the opt-in per-channel asymmetric quantizer (not the reference scheme)")
    ap.add_argument("--ctas", type=int, default=None,
                    help="split-kernel grid: default persistent (resident CTAs), 0 = one CTA per 256-row slice")
    ap.add_argument("--layers", type=int, default=None, help="override layer count (debug only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
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
    """--impl reference: the oracle port on host cores, rank 0 only."""
    global_batch = cfg["batch"] * world
    units_per_step = cfg["layers"] * global_batch * (cfg["kv_heads"] // world) * world
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
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic N(0,1) K/V rounded to fp16; oracle units encoded once per worker",
        "config": {"workload": cfg["workload"], "global_batch": global_batch, "context": cfg["T"],
                   "kv_bits": cfg["bits"], "layers": cfg["layers"], "kv_heads": cfg["kv_heads"], "g": cfg["g"]},
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


def run_ours(args, cfg):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2405_12591_b200.attention import DecodeKvCache

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    layers = args.layers or cfg["layers"]
    kv_heads, g, bits, T = cfg["kv_heads"], cfg["g"], cfg["bits"], cfg["T"]
    if kv_heads % world:
        raise SystemExit(f"{kv_heads} kv heads do not shard over {world} GPUs")
    global_batch = cfg["batch"] * world
    local_heads = kv_heads // world
    units = global_batch * local_heads  # (sequence, local kv head) pairs on this rank
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

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # steady state: a partly filled fp16 tail, appended through the public API
    for layer in range(layers):
        for _ in range(args.tail):
            cache.append_token(layer, kn[layer], vn[layer])
    torch.cuda.synchronize()
    appended = args.tail + args.warmup + args.steps + 1 + max(3, args.warmup // 2) + max(3, args.steps // 2)
    if appended + 1 >= chunk_len:
        raise SystemExit("steps too large: the tail would seal a chunk inside the timed region")

    # ---- device-resident timed region ----------------------------------------------
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            step()
        ev1.record()
        torch.cuda.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    value = global_batch / (ms / 1e3)

    # ---- split-kernel launches alone, for the roofline -------------------------------
    kstarts = [torch.cuda.Event(enable_timing=True) for _ in range(layers)]
    kends = [torch.cuda.Event(enable_timing=True) for _ in range(layers)]
    durs = []
    for rep in range(3):
        for layer in range(layers):
            kstarts[layer].record()
            cache.launch(layer, q[layer], out[layer], phases=1)
            kends[layer].record()
        torch.cuda.synchronize()
        if rep:
            durs += [kstarts[i].elapsed_time(kends[i]) for i in range(layers)]
    kern_ms = statistics.mean(durs)
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
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16",
        "data": "synthetic: per-layer K/V ~ N(0,1) fp16 compressed by the K3 write path; q/k/v rows ~ N(0,1) fp16",
        "config": {"workload": cfg["workload"], "global_batch": global_batch, "seq_len": T, "context": T,
                   "kv_bits": bits, "tail_tokens": args.tail, "quantizer": "per-channel asymmetric (opt-in)" if args.asym else "per-tensor symmetric (reference)",
                   "layers": layers, "kv_heads": kv_heads, "g": g,
                   "parallelism": f"kv-head shards x{world}", "units_per_gpu": units, "chunk_b": cache._layers[0].args.chunk_b,
                   "split_ctas": cache.split_ctas, "kernel_g": cache._layers[0].kernel_g,
                   "head_groups": g // cache._layers[0].kernel_g,
                   "split_path": {0: "mma.sync", 1: "tcgen05", 2: "tcgen05-gqa"}[cache._layers[0].args.path],
                   "l2": f"inputs > L2: {step_bytes / 1e9:.2f} GB streamed per step per GPU"},
        "hbm_gbs_step": step_bytes / (ms / 1e3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "kernel": {0: "decode_attn_kernel", 1: "decode_attn_tc_kernel", 2: "decode_attn_gqa_kernel"}[cache._layers[0].args.path],
                     "bytes_per_launch": kern_bytes,
                     "launch_ms": kern_ms, "peak_kind": peak_kind},
        "memory_per_token_vs_fp16": actual_bytes / fp16_bytes,
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
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            run_reference(args, cfg, world)
        return
    run_ours(args, cfg)


if __name__ == "__main__":
    main()
