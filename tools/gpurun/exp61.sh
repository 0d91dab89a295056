# cuBLAS M=16 decode GEMM launch config (grid / smem / DRAM) for comparison with the TBIK GEMM
mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 \
    -o gpurun_out/e61_cublas_m16 python tools/prof_shape.py 16 14336 4096 3 --cublas > gpurun_out/e61_fc.log 2>&1
ncu --set full --clock-control none -k regex:nvjet -s 2 -c 1 \
    -o gpurun_out/e61_cublas_m64 python tools/prof_shape.py 64 14336 4096 3 --cublas > gpurun_out/e61_fc64.log 2>&1
