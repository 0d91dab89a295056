#!/bin/bash
# r02: R1 variant (level 1 in registers, 8 stages) -- a 60 s single-call probe first, then the
# GEMM tests and the A/B at the bench shape and mid-M.  Timeouts sum well below the gpurun limit.
mkdir -p gpurun_out
timeout 60 python tools/ab_knobs.py 4096 14336 4096 > gpurun_out/r02_r1_probe.txt 2>&1; rc=$?
echo "probe rc=$rc" >> gpurun_out/r02_r1_probe.txt
if [ $rc -ne 0 ]; then cat gpurun_out/r02_r1_probe.txt; exit 1; fi
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_leaf_adversarial.py -q -x > gpurun_out/r02_r1_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r02_r1_tests.log
timeout 300 python tools/ab_knobs.py > gpurun_out/r02_r1_ab.txt 2>&1
cat gpurun_out/r02_r1_probe.txt; tail -3 gpurun_out/r02_r1_tests.log; cat gpurun_out/r02_r1_ab.txt
