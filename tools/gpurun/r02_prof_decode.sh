#!/bin/bash
# r02: ncu of the TP = 8 decode shard GEMM (skinny kernel vs cuBLAS).
mkdir -p gpurun_out
tag=${1:-r02_pd}
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"tc_skinny|nvjet|gemm|splitK" -s 2 -c 4 \
  -o gpurun_out/${tag} python tools/prof_decode.py 16 1792 4096 7 3 > gpurun_out/${tag}.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}.log
tail -3 gpurun_out/${tag}.log
