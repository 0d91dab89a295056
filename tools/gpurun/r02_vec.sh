#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -m gpu -k "skinny or schedule" > gpurun_out/r02_vec_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02_vec_tests.log
tail -n 3 gpurun_out/r02_vec_tests.log
bash tools/gpurun/r02_sk_trace.sh > /dev/null 2>&1; cp gpurun_out/r02_sk_trace.txt gpurun_out/r02_sk_trace_vec.txt; grep -v "^==" gpurun_out/r02_sk_trace_vec.txt | cut -c1-200
timeout 400 python tools/decode_bench.py 1 16 64 128 > gpurun_out/r02_vec_decode.txt 2>&1
cat gpurun_out/r02_vec_decode.txt | cut -c1-450
