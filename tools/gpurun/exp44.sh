mkdir -p gpurun_out
S="4096 14336 4096 4096 4096 28672"
for cfg in "0 0" "0 1" "1 0" "1 1" "5 0" "5 1"; do set -- $cfg
  TBIK_TC_DEBUG=$1 TBIK_TC_DEEP=$2 timeout 120 python tools/ab_shape.py "dbg=$1 deep=$2" $S
done > gpurun_out/e44.txt 2>&1
