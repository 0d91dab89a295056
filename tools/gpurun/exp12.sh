mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_tree_gemm -s 2 -c 1 -o gpurun_out/e12_m16 python tools/prof_shape.py 16 14336 4096 3 > gpurun_out/e12_a.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 -o gpurun_out/e12_m16_cublas python tools/prof_shape.py 16 14336 4096 3 --cublas > gpurun_out/e12_b.log 2>&1
TBIK_TC_DEBUG=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_tree_gemm -s 2 -c 1 -o gpurun_out/e12_nomerge python tools/prof_shape.py 4096 14336 4096 3 > gpurun_out/e12_c.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_tree_gemm -s 2 -c 1 -o gpurun_out/e12_full python tools/prof_shape.py 4096 14336 4096 3 > gpurun_out/e12_d.log 2>&1
