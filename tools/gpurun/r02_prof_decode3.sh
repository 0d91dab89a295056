#!/bin/bash
# r02: source-level stall sampling (32-cycle interval) of the skinny kernel on the TP=8 decode shard.
mkdir -p gpurun_out
timeout 300 ncu --section SourceCounters --section WarpStateStats --warp-sampling-interval 0 --clock-control none --import-source on \
  -k regex:tc_skinny -s 5 -c 1 -o gpurun_out/r02s4_pd3 python tools/prof_decode.py 16 1792 4096 7 8 > gpurun_out/r02s4_pd3.log 2>&1
tail -2 gpurun_out/r02s4_pd3.log
