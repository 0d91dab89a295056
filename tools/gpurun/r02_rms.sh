#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_rowops.py -q -x -m gpu > gpurun_out/r02_rms_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02_rms_tests.log
tail -n 2 gpurun_out/r02_rms_tests.log
timeout 300 python tools/rowops_bench.py > gpurun_out/r02_rms_bench.txt 2>&1
cat gpurun_out/r02_rms_bench.txt | head -30
