#!/bin/bash
# r02: 16-warp tcgen05 attention (4 threads per row, S double-buffered in TMEM): tests + timing vs mma.sync.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_model.py -q -x -k "attention" > gpurun_out/tc5b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/tc5b_tests.log
bash tools/gpurun/r02_tc5_perf.sh > gpurun_out/tc5b_perf.txt 2>&1
tail -3 gpurun_out/tc5b_tests.log; cat gpurun_out/tc5b_perf.txt
