#!/bin/bash
mkdir -p gpurun_out
( for ks in 64 128; do
  for shape in "16 1792 4096 7" "128 1792 4096 7" "16 3584 4096 7"; do
    echo "== ks=$ks shape=$shape"
    timeout 60 python tools/prof_decode.py $shape 3 --knob sk_ks=$ks --knob sk_trace=1 2>&1 | grep sk_trace | tail -1 | cut -c1-250
  done
done ) > gpurun_out/r02_sk_trace2.txt 2>&1
cat gpurun_out/r02_sk_trace2.txt
