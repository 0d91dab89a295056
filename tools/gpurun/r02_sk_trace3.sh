#!/bin/bash
# r02: skinny phase clocks on the cluster (K-split) shapes + bits + decode table.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -m gpu -k "skinny or schedule" > gpurun_out/r02_t3_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02_t3_tests.log
tail -n 2 gpurun_out/r02_t3_tests.log
( for shape in "16 1792 4096 7" "16 3584 4096 7" "16 7168 4096 7" "128 3584 4096 7" "16 14336 4096 0"; do
    echo "== shape=$shape"
    timeout 60 python tools/prof_decode.py $shape 3 --knob sk_trace=1 2>&1 | grep sk_trace | tail -1 | cut -c1-250
  done ) > gpurun_out/r02_sk_trace3.txt 2>&1
cat gpurun_out/r02_sk_trace3.txt
timeout 400 python tools/decode_bench.py 1 16 64 128 > gpurun_out/r02_t3_decode.txt 2>&1
grep graph gpurun_out/r02_t3_decode.txt | awk -F'|' '{print $1 "|" $3 "|" $NF}'
