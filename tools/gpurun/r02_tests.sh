#!/bin/bash
# r02: the full GPU suite (+ the adversarial leaf tests printed).
mkdir -p gpurun_out
tag=${1:-r02_tests}
timeout 2400 python -m pytest tests -m gpu -x -q -rs > gpurun_out/${tag}.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}.log
timeout 600 python -m pytest tests/test_gpu_leaf_adversarial.py -q -s -k adversarial > gpurun_out/${tag}_adv.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
tail -5 gpurun_out/${tag}.log; cat gpurun_out/${tag}_adv.log | tail -20; tail -2 gpurun_out/${tag}_smoke.log
