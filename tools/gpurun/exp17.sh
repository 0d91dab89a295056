mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/e17_fwd_launches.csv python tools/forward_once.py > gpurun_out/e17_fwd.log 2>&1
