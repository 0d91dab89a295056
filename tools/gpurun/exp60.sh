# small-M (decode regime) diagnosis: launch list + full ncu of the M=16 TBIK GEMM and cuBLAS
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/e60_build.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e60_launches.csv \
    python tools/prof_shape.py 16 14336 4096 3 --cublas > gpurun_out/e60_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_tree_gemm -s 2 -c 1 \
    -o gpurun_out/e60_tc_m16 python tools/prof_shape.py 16 14336 4096 3 > gpurun_out/e60_f.log 2>&1
ncu --set full --clock-control none -k regex:"gemm|Kernel|nvjet" -s 2 -c 1 \
    -o gpurun_out/e60_cublas_m16 python tools/prof_shape.py 16 14336 4096 3 --cublas > gpurun_out/e60_fc.log 2>&1
ls -la gpurun_out
