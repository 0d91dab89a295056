mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size,launch__cluster_size --clock-control none --csv --log-file gpurun_out/e83_launches.csv \
    python tools/prof_shape.py 16 1792 4096 3 --cublas > gpurun_out/e83.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:skinny -s 2 -c 1 \
    -o gpurun_out/e83_skinny_tp8 python tools/prof_shape.py 16 1792 4096 3 > gpurun_out/e83_f.log 2>&1
