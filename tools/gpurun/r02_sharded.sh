#!/bin/bash
# r02: real-TP sharded forward (W processes on one GPU) + the collective tests.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_sharded_forward.py tests/test_gpu_collective.py -x -q -s > gpurun_out/r02_sharded.log 2>&1
echo "rc=$?" >> gpurun_out/r02_sharded.log
tail -40 gpurun_out/r02_sharded.log
