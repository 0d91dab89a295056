#!/bin/bash
# r02 final evidence: default bench line (timed by wall clock too), ncu --set full of the bench
# kernel, the bench launch list, the reference arm.
mkdir -p gpurun_out
tag=${1:-r02_final}
start=$(date +%s)
timeout 1200 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "rc=$? wall=$(( $(date +%s) - start ))s" >> gpurun_out/${tag}_bench.err
timeout 420 ncu --set full --clock-control none --import-source on -k regex:"tc_w192|tc_tree_gemm" -s 2 -c 1 \
  -o gpurun_out/${tag}_tc python tools/prof_shape.py 4096 14336 4096 3 > gpurun_out/${tag}_tc.log 2>&1
echo "ncu full rc=$?" >> gpurun_out/${tag}_tc.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-forward \
  > gpurun_out/${tag}_ncu_bench.log 2>&1
echo "launch list rc=$?" >> gpurun_out/${tag}_ncu_bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "rc=$?" >> gpurun_out/${tag}_ref.err
tail -n 2 gpurun_out/${tag}_bench.err gpurun_out/${tag}_tc.log gpurun_out/${tag}_ncu_bench.log gpurun_out/${tag}_ref.err
