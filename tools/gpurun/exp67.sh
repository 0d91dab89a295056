mkdir -p gpurun_out
for M in 64 128; do
ncu --set full --clock-control none --import-source on -k regex:skinny -s 2 -c 1 \
    -o gpurun_out/e67_skinny_m$M python tools/prof_shape.py $M 14336 4096 3 > gpurun_out/e67_f$M.log 2>&1
done
