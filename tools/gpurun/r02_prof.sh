#!/bin/bash
# r02: ncu --set full capture of the bench-shape tree GEMM (source-level stall sampling) and
# the launch list of the bench step.  Per-command timeouts sum below the gpurun limit.
mkdir -p gpurun_out
tag=${1:-r02_prof}
timeout 420 ncu --set full --clock-control none --import-source on -k regex:tc_tree_gemm -s 2 -c 1 \
  -o gpurun_out/${tag}_tc python tools/prof_shape.py 4096 14336 4096 3 > gpurun_out/${tag}_tc.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${tag}_tc.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-forward \
  > gpurun_out/${tag}_ncu_bench.log 2>&1
echo "launch list rc=$?" >> gpurun_out/${tag}_ncu_bench.log
tail -2 gpurun_out/${tag}_tc.log gpurun_out/${tag}_ncu_bench.log
