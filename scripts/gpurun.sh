#!/bin/bash
# Rebuilds libepk.so (nvcc cross-compile) and runs "$@" on a B200 via gpurun.
cd "$(dirname "$0")/.."
python paper_2509_17396_b200/_build.py > /tmp/epk_build.log 2>&1 || { grep -v "^/usr/local/cuda/bin/nvcc" /tmp/epk_build.log | tail -30; exit 1; }
exec /usr/local/graft/bin/gpurun --timeout "${GPU_TIMEOUT:-1200}" -- "$@"
