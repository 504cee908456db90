#!/bin/bash
# build a -DDQ_ATTN_WARP_TRACE copy of the library and run scripts/warp_trace.py with it
set -e
rm -rf /tmp/wtrace && mkdir -p /tmp/wtrace && cp -r paper_2405_12591_b200 include scripts /tmp/wtrace/
cd /tmp/wtrace
python - <<'PY'
import sys
sys.path.insert(0, ".")
from paper_2405_12591_b200 import build as B
B.FLAGS.append("-DDQ_ATTN_WARP_TRACE")
import os
if os.environ.get("EXTRA"): B.FLAGS += os.environ["EXTRA"].split()
B.build(force=True)
PY
python scripts/warp_trace.py
