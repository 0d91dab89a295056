mkdir -p gpurun_out
S="4096 14336 4096 2048 14336 8192"
for d in 1 65; do for st in 4 5; do
  TBIK_TC_WIDE=1 TBIK_TC_WIDE_STAGES=$st TBIK_TC_DEBUG=$d timeout 120 python tools/ab_shape.py "wide st=$st dbg=$d" $S
done; done > gpurun_out/e48.txt 2>&1
