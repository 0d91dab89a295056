#!/bin/bash
# r02: ncu --set full of the 256x128 and 256x256 tree GEMMs and cuBLAS at the bench shape.
mkdir -p gpurun_out
tag=${1:-r02_prof_wide}
shift
for spec in "narrow:tc_wide=0" "wide:tc_wide=1" "$@"; do
  name=${spec%%:*}; knob=${spec#*:}
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_ -s 1 -c 1 \
    -o gpurun_out/${tag}_${name} python tools/prof_shape.py 4096 14336 4096 2 --knob $knob > gpurun_out/${tag}_${name}.log 2>&1
  echo "$name rc=$?" >> gpurun_out/${tag}_${name}.log
done
timeout 300 ncu --set full --clock-control none -k regex:nvjet -s 1 -c 1 \
  -o gpurun_out/${tag}_cublas python tools/prof_shape.py 4096 14336 4096 2 --cublas > gpurun_out/${tag}_cublas.log 2>&1
tail -n 2 gpurun_out/${tag}_*.log
