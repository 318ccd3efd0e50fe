#!/bin/bash
# Guard-band memory check (stands in for compute-sanitizer memcheck, which the
# GPU pool does not allow): build the library with -DPS_CANARY (64 KB of 0xA5
# after every context allocation, verified at free and at the end), run the
# kernel-family driver and the GPU test suite against it, report overruns.
set -e
cd "$(dirname "$0")/.."
LIB=paper_1412_7466_b200/libperiscat_b200_canary.so
[ -f "$LIB" ] || python -m paper_1412_7466_b200.build -DPS_CANARY --out=$LIB
export PS_LIB=$PWD/$LIB
python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1412_7466_b200 import _lib
lib = _lib.load()
print("canary selftest (deliberate 1-byte overrun seen):", lib.ps_canary_selftest())
PY
python tools/sanitize_run.py
python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
from paper_1412_7466_b200 import _lib
print("canary violations after the kernel-family driver:", _lib.load().ps_canary_check())
PY
PS_CANARY_CHECK=1 python -m pytest tests -m gpu -q -s -p no:cacheprovider \
    --deselect tests/test_gpu_krylov.py::test_sharded_schur_and_gmres_multiprocess_one_gpu 2>&1 \
    | grep -E "passed|failed|canary"
