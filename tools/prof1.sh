set -x
mkdir -p gpurun_out
./tools/micro/tmem_ld_bw > gpurun_out/p1_tmem.txt 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_tree_gemm -s 2 -c 1 -o gpurun_out/p1_tc python tools/prof_shape.py 4096 14336 4096 3 > gpurun_out/p1_tc.log 2>&1
timeout 300 ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 -o gpurun_out/p1_cublas python tools/prof_shape.py 4096 14336 4096 3 --cublas > gpurun_out/p1_cublas.log 2>&1
timeout 300 python tools/rowops_bench.py > gpurun_out/p1_rowops.json 2> gpurun_out/p1_rowops.err
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:rmsnorm|ms_group|ms_rows|merge|finish|allreduce' -c 8 -o gpurun_out/p1_rowops python tools/rowops_bench.py > gpurun_out/p1_rowops_ncu.log 2>&1
ls -la gpurun_out
