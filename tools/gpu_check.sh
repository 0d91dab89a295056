#!/bin/bash
# One GPU-box pass: GPU tests, smoke, default bench, ncu launch list of the bench step.
# usage (from the repo root, via gpurun): bash tools/gpu_check.sh [tag]
tag=${1:-check}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-forward \
  > gpurun_out/${tag}_ncu_bench.log 2>&1
tail -3 gpurun_out/${tag}_pytest.log gpurun_out/${tag}_smoke.log
