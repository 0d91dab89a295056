#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_model.py -q -x -m gpu -k "attention" > gpurun_out/r02_attn_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02_attn_tests.log
tail -n 2 gpurun_out/r02_attn_tests.log
timeout 300 python tools/attn_sv1_ab.py 2>&1 | tail -5
