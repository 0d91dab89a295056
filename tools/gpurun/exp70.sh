mkdir -p gpurun_out
timeout 600 python tools/midm_sweep.py > gpurun_out/e70_midm.txt 2>&1; echo "rc=$?" >> gpurun_out/e70_midm.txt
