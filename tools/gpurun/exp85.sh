mkdir -p gpurun_out
timeout 600 python tools/midm_sweep.py --mc > gpurun_out/e85_mc.txt 2>&1; echo "rc=$?" >> gpurun_out/e85_mc.txt
