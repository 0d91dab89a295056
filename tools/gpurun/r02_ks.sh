#!/bin/bash
# r02: skinny kernel with 128-row W boxes (sk_ks) -- bits vs the wide kernel, decode timings.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -m gpu -k "skinny" > gpurun_out/r02_ks_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02_ks_tests.log
tail -n 3 gpurun_out/r02_ks_tests.log
timeout 900 python tools/decode_bench.py 1 16 64 128 > gpurun_out/r02_ks_decode.txt 2>&1
cat gpurun_out/r02_ks_decode.txt | cut -c1-400
