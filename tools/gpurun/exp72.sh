mkdir -p gpurun_out
timeout 600 python tools/ab_debug.py > gpurun_out/e72_ab.txt 2>&1; echo "rc=$?" >> gpurun_out/e72_ab.txt
