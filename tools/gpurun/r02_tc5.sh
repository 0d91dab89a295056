#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_model.py -q -x -m gpu -k "attention_tc_invariance" > gpurun_out/r02_tc5_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02_tc5_tests.log
tail -n 25 gpurun_out/r02_tc5_tests.log | cut -c1-250
