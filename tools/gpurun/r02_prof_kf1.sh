#!/bin/bash
# r02: ncu --set full of the k_first = 1 shape (o_proj M=K=N=4096): where does the MMA issuer wait?
mkdir -p gpurun_out
timeout 420 ncu --set full --clock-control none --import-source on -k regex:tc_tree_gemm -s 2 -c 1 \
  -o gpurun_out/r02_prof_kf1 python tools/prof_shape.py 4096 4096 4096 3 > gpurun_out/r02_prof_kf1.log 2>&1
echo "rc=$?" >> gpurun_out/r02_prof_kf1.log
