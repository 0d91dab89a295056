mkdir -p gpurun_out
S="4096 14336 4096"
for d in 0 4 8 16 24 32 56; do
  TBIK_TC_WIDE=1 TBIK_TC_WIDE_STAGES=5 TBIK_TC_DEBUG=$d timeout 120 python tools/ab_shape.py "wide st=5 dbg=$d" $S
done > gpurun_out/e47.txt 2>&1
