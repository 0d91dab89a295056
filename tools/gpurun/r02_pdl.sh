#!/bin/bash
# r02: skinny kernel with PDL + no lone-CTA cluster barriers: bits, phase clocks, decode timings.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x -m gpu -k "skinny" > gpurun_out/r02_pdl_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02_pdl_tests.log
tail -n 3 gpurun_out/r02_pdl_tests.log
bash tools/gpurun/r02_sk_trace.sh > /dev/null 2>&1; cp gpurun_out/r02_sk_trace.txt gpurun_out/r02_sk_trace_pdl.txt; cat gpurun_out/r02_sk_trace_pdl.txt
timeout 900 python tools/decode_bench.py 1 16 64 128 > gpurun_out/r02_pdl_decode.txt 2>&1
cat gpurun_out/r02_pdl_decode.txt | cut -c1-450
