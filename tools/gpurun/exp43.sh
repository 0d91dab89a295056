mkdir -p gpurun_out
TBIK_TC_WIDE=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:wide -s 2 -c 1 -o gpurun_out/e43_wide python tools/prof_shape.py 4096 14336 4096 3 > gpurun_out/e43_wide.log 2>&1
TBIK_TC_MC=1 timeout 300 ncu --set full --clock-control none -k regex:tc_tree -s 2 -c 1 -o gpurun_out/e43_mc python tools/prof_shape.py 4096 14336 4096 3 > gpurun_out/e43_mc.log 2>&1
