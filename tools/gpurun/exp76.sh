mkdir -p gpurun_out
for K in 4096 14336; do
ncu --set full --clock-control none --import-source on -k regex:tc_tree_gemm -s 2 -c 1 \
    -o gpurun_out/e76_tc_k$K python tools/prof_shape.py 4096 $K 4096 3 > gpurun_out/e76_k$K.log 2>&1
done
