#!/bin/bash
mkdir -p gpurun_out
timeout 600 python tools/fwd_profile.py 8 4 256 > gpurun_out/r02_fwdprof.txt 2>&1
echo "rc=$?" >> gpurun_out/r02_fwdprof.txt
for shp in "1024 4096 6144" "1024 4096 4096" "1024 4096 28672" "1024 14336 4096" "1024 4096 128256"; do
  MID=1 timeout 300 python tools/wide_check.py time $shp 2>&1 | tail -1
done > gpurun_out/r02_fwd_shapes.txt 2>&1
head -40 gpurun_out/r02_fwdprof.txt; cat gpurun_out/r02_fwd_shapes.txt
