#!/bin/bash
# Round-end evidence pass on one B200 (run via gpurun from the repo root):
# GPU tests, smoke, the default bench line, the launch list of the bench step,
# one ncu --set full capture of the dominant kernel, C5 row reductions.
tag=${1:-final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 1200 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu --no-forward \
  > gpurun_out/${tag}_ncu_bench.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_tree_gemm -s 2 -c 1 \
  -o gpurun_out/${tag}_tc python tools/prof_shape.py 4096 14336 4096 3 > gpurun_out/${tag}_tc.log 2>&1
