mkdir -p gpurun_out
timeout 600 python tools/midm_sweep.py --epi > gpurun_out/e73_epi.txt 2>&1; echo "rc=$?" >> gpurun_out/e73_epi.txt
