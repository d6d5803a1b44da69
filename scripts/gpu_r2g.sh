#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -k "sensitiv or kmeans" > gpurun_out/t.log 2>&1; echo "rc=$?" >> gpurun_out/t.log
grep -E "passed|failed|Error|assert" gpurun_out/t.log | head -30
timeout 300 ./tests/cpp/_build/test_dropin 2>&1 | tail -5
timeout 300 ./tests/cpp/_build/test_build 2>&1 | tail -8
timeout 300 python scripts/time_k4k5.py 2>&1 | tail -12
