#!/bin/bash
# r02: skinny CTA-pair split of a single leaf group: bits, phase clocks, decode table.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -m gpu -k "skinny or schedule" > gpurun_out/r02_pair_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02_pair_tests.log
tail -n 4 gpurun_out/r02_pair_tests.log
( for shape in "128 1792 4096 7" "64 1792 4096 7"; do
    echo "== shape=$shape"
    timeout 60 python tools/prof_decode.py $shape 3 --knob sk_trace=1 2>&1 | grep sk_trace | tail -2 | cut -c1-250
  done ) > gpurun_out/r02_pair_trace.txt 2>&1
cat gpurun_out/r02_pair_trace.txt
timeout 400 python tools/decode_bench.py 1 16 > gpurun_out/r02_pair_decode.txt 2>&1
grep graph gpurun_out/r02_pair_decode.txt | awk -F'|' '{print $1 "|" $3 "|" $(NF-1) "|" $NF}'
