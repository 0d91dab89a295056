#!/bin/bash
# r02: 256x256 pair-tile kernel -- bit equality vs the 256x128 kernel, then timings.
mkdir -p gpurun_out
tag=${1:-r02_wide}
timeout 300 python tools/wide_check.py check > gpurun_out/${tag}_check.txt 2>&1; rc=$?
echo "check rc=$rc" >> gpurun_out/${tag}_check.txt
cat gpurun_out/${tag}_check.txt
if [ $rc -ne 0 ]; then exit 1; fi
timeout 400 python tools/wide_check.py time > gpurun_out/${tag}_time.txt 2>&1; echo "time rc=$?" >> gpurun_out/${tag}_time.txt
cat gpurun_out/${tag}_time.txt
