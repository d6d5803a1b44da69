#!/bin/bash
# Builds locally (nvcc cross-compile) and runs the CPU suite's ABI check
# before spending a gpurun call; then runs "$@" on a B200 via gpurun.
set -e
cd "$(dirname "$0")/.."
python paper_2509_17396_b200/_build.py > /tmp/epk_build.log 2>&1 || { grep -v "^/usr/local/cuda/bin/nvcc" /tmp/epk_build.log | tail -30; exit 1; }
python -m pytest -q tests/test_abi.py > /tmp/epk_abi.log 2>&1 || { tail -20 /tmp/epk_abi.log; exit 1; }
TO=${GPU_TIMEOUT:-900}
exec /usr/local/graft/bin/gpurun --timeout "$TO" -- "$@"
