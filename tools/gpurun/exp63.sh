mkdir -p gpurun_out
timeout 300 python tools/decode_bench.py > gpurun_out/e63_decode.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:skinny -s 2 -c 1 \
    -o gpurun_out/e63_skinny_m16 python tools/prof_shape.py 16 14336 4096 3 > gpurun_out/e63_f.log 2>&1
