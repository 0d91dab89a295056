#!/bin/bash
# r02: drop-in boundary (C++ headers, reference runner.cpp on the B200 lib, local group,
# baseline layers) + the process-group collective tests (ragged K).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_boundary.py tests/test_gpu_cpp_api.py tests/test_gpu_collective.py -x -q -s > gpurun_out/r02_boundary.log 2>&1
echo "rc=$?" >> gpurun_out/r02_boundary.log
tail -60 gpurun_out/r02_boundary.log
