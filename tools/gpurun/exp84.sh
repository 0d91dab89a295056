mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max --clock-control none --csv --log-file gpurun_out/e84_tiny.csv \
    python tools/prof_shape.py 1 256 64 3 --cublas > gpurun_out/e84.log 2>&1
ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max --clock-control none --csv --log-file gpurun_out/e84_tp8.csv \
    python tools/prof_shape.py 16 1792 4096 3 --cublas > gpurun_out/e84b.log 2>&1
