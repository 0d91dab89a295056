#!/bin/bash
# r02: skinny TP = 8 shard (M=16 K=1792 N=4096) kernel durations, 64- vs 128-row W boxes, warm L2.
mkdir -p gpurun_out
for ks in 64 128; do
  timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,l1tex__m_xbar2l1tex_read_bytes.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum \
    --clock-control none --cache-control none -k regex:"tc_skinny|nvjet" -c 12 --csv python tools/prof_decode.py 16 1792 4096 7 6 --knob sk_ks=$ks > gpurun_out/r02_ks_prof_$ks.csv 2>&1
done
timeout 300 ncu --set full --clock-control none --cache-control none --import-source on -k regex:tc_skinny -s 5 -c 1 -o gpurun_out/r02_ks128 python tools/prof_decode.py 16 1792 4096 7 8 > /dev/null 2>&1
for ks in 64 128; do grep -E "gpu__time_duration" gpurun_out/r02_ks_prof_$ks.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | cut -c1-120 | tail -12; done
