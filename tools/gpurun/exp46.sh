mkdir -p gpurun_out
S="4096 14336 4096 1024 14336 4096"
for d in 0 1 4; do
  TBIK_TC_WIDE=1 TBIK_TC_WIDE_STAGES=5 TBIK_TC_DEBUG=$d timeout 120 python tools/ab_shape.py "wide st=5 dbg=$d" $S
done > gpurun_out/e46.txt 2>&1
TBIK_TC_WIDE=1 TBIK_TC_WIDE_STAGES=5 timeout 300 ncu --set full --clock-control none --import-source on -k regex:wide -s 2 -c 1 -o gpurun_out/e46_wide python tools/prof_shape.py 4096 14336 4096 3 > gpurun_out/e46_wide.log 2>&1
