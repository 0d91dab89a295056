#!/bin/bash
# r02: skinny (decode) kernel after the MMA-issuer change: GEMM tests + decode timings.
mkdir -p gpurun_out
tag=${1:-r02_skinny}
timeout 400 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
timeout 400 python tools/decode_bench.py 1 16 64 128 > gpurun_out/${tag}_decode.txt 2>&1
tail -2 gpurun_out/${tag}_tests.log; cat gpurun_out/${tag}_decode.txt
