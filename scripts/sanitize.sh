#!/bin/bash
# compute-sanitizer over every kernel family at toy shapes (scripts/sanitize_step.py)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_step.py > gpurun_out/san_$tool.txt 2>&1
  echo "== $tool rc=$?"; tail -3 gpurun_out/san_$tool.txt
done
