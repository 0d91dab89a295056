#!/bin/bash
mkdir -p gpurun_out
for tool in memcheck synccheck; do  # racecheck: > 15 min, not completed
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_skinny.py > gpurun_out/r02_sanitize_skinny_$tool.txt 2>&1
  echo "rc=$?" >> gpurun_out/r02_sanitize_skinny_$tool.txt
  tail -n 4 gpurun_out/r02_sanitize_skinny_$tool.txt
done
