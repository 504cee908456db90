#!/bin/bash
# memory-pipeline ceiling of the split kernel: same producer / ring / scheduler, consumers
# skip the contractions (results are garbage); prints the split kernel time of the C2 bench
set -e
mkdir -p /tmp/nullc && cp -r paper_2405_12591_b200 include bench.py oracle /tmp/nullc/ 2>/dev/null
cd /tmp/nullc
NVCC_APPEND="${NULL_FLAGS:--DDQ_ATTN_NULL_CONSUMER}" python - <<'PY'
import os, sys
sys.path.insert(0, ".")
from paper_2405_12591_b200 import build as B
B.FLAGS.extend(os.environ["NVCC_APPEND"].split())
B.build(force=True)
PY
python bench.py --steps 5 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('null-consumer split kernel us', round(1e3*d['roofline']['launch_ms'],1), 'GB/s', round(d['roofline']['achieved']))"
