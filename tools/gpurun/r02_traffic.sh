#!/bin/bash
# r02: cold-cache DRAM bytes per call for every roofline the bench line reports.
mkdir -p gpurun_out
tag=${1:-r02_traffic}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --print-units base \
  --clock-control none --kernel-name-base demangled -k regex:tbik_b200 --csv --log-file gpurun_out/${tag}.csv \
  python tools/traffic_capture.py > gpurun_out/${tag}.log 2>&1
echo "rc=$?" >> gpurun_out/${tag}.log
python tools/traffic_reduce.py gpurun_out/${tag}.csv gpurun_out/${tag}.log gpurun_out/${tag}.json | head -60
