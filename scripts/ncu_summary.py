#!/usr/bin/env python
"""Summarise an ncu report: key raw metrics + per-source-line stall/instruction shares.

    python scripts/ncu_summary.py gpurun_out/prof_attn_v2.ncu-rep [--lines 25]
"""
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    nlines = int(sys.argv[sys.argv.index("--lines") + 1]) if "--lines" in sys.argv else 25
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "raw", "--csv"]))))
    hdr, units, vals = rows[0], rows[1], rows[2]
    print("kernel:", vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?")
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            print(f"  {m:70s} {vals[i]:>16s} {units[i]}")
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]))))
    h = rows[2]
    i_inst = h.index("Instructions Executed")
    agg = collections.defaultdict(lambda: [0, 0])
    cur = None
    for r in rows[3:]:
        if r and r[0]:
            cur = (r[0], r[1].strip()[:90])
            continue
        if len(r) > i_inst and r[2] not in ("...", ""):
            try:
                agg[cur][0] += int(r[4] or 0)
                agg[cur][1] += int(r[i_inst] or 0)
            except ValueError:
                pass
    ts = sum(v[0] for v in agg.values()) or 1
    ti = sum(v[1] for v in agg.values()) or 1
    print(f"stall samples {ts}, instructions {ti}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:nlines]:
        print(f"  {100 * v[0] / ts:5.1f}% stall {100 * v[1] / ti:5.1f}% inst  L{k[0]}: {k[1]}")


if __name__ == "__main__":
    main()


def opcode_mix(rep, top=25):
    """Executed warp-instructions per SASS opcode."""
    rows = list(csv.reader(io.StringIO(run([rep, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = rows[1]
    i_src, i_inst = h.index("Source"), h.index("Instructions Executed")
    agg = collections.Counter()
    for r in rows[2:]:
        if len(r) > i_inst and r[i_inst] not in ("", "-"):
            toks = r[i_src].split()
            if not toks:
                continue
            op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
            agg[op.split(".")[0]] += int(r[i_inst])
    tot = sum(agg.values()) or 1
    for op, n in agg.most_common(top):
        print(f"  {op:10s} {n:12d} {100 * n / tot:5.1f}%")
