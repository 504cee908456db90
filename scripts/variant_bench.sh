#!/bin/bash
# A/B of a compile-time variant of the kernels on one box: bench of this tree as built,
# then of a copy built with extra nvcc flags.
#   VFLAGS="-DDQ_ATTN_WARPS=16 ..." bash scripts/variant_bench.sh [bench args]
set -e
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline $*"
show() { python -c "import json,sys; d=json.loads(sys.stdin.read()); print(sys.argv[1], 'ms/step', round(d['ms_per_step'],3), 'split_us', round(1e3*d['roofline']['launch_ms'],1), 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']))" "$1"; }
$B 2>/dev/null | show base
rm -rf /tmp/variant && mkdir -p /tmp/variant && cp -r paper_2405_12591_b200 include bench.py oracle MEASURED_PEAKS.json profiles /tmp/variant/ 2>/dev/null || true
cd /tmp/variant
VFLAGS="$VFLAGS" python - <<'PY'
import os, sys
sys.path.insert(0, ".")
from paper_2405_12591_b200 import build as B
B.FLAGS.extend(os.environ["VFLAGS"].split())
B.build(force=True)
PY
$B 2>/dev/null | show variant
python -m pytest -q -x -p no:cacheprovider /root/repo/tests/test_gpu_attention.py -k "prefill_only and 4-1-4096" --rootdir /tmp/variant 2>&1 | tail -1 || true
