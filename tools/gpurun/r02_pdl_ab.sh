#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -m gpu > gpurun_out/r02_pdl_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02_pdl_tests.log
tail -n 2 gpurun_out/r02_pdl_tests.log
timeout 600 python tools/pdl_ab.py > gpurun_out/r02_pdl_ab.txt 2>&1; cat gpurun_out/r02_pdl_ab.txt
timeout 900 python tools/forward_bench.py > gpurun_out/r02_pdl_fwd.txt 2>&1; tail -5 gpurun_out/r02_pdl_fwd.txt | cut -c1-300
