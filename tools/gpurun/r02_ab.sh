#!/bin/bash
# r02: quick correctness + A/B after a GEMM change (GEMM tests, schedule A/B, short bench).
mkdir -p gpurun_out
tag=${1:-r02_ab}
timeout 60 python tools/ab_knobs.py 4096 14336 4096 > gpurun_out/${tag}_probe.txt 2>&1; rc=$?
echo "probe rc=$rc" >> gpurun_out/${tag}_probe.txt
if [ $rc -ne 0 ]; then cat gpurun_out/${tag}_probe.txt; exit 1; fi
timeout 500 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_leaf_adversarial.py tests/test_gpu_collective.py -q -x > gpurun_out/${tag}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_tests.log
timeout 200 python tools/ab_knobs.py > gpurun_out/${tag}_ab.txt 2>&1
timeout 200 python bench.py --no-sweep --no-forward --no-cpu > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -2 gpurun_out/${tag}_tests.log; cat gpurun_out/${tag}_ab.txt; head -c 400 gpurun_out/${tag}_bench.json
