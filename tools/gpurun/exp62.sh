mkdir -p gpurun_out
timeout 300 python tools/skinny_check.py --time-only > gpurun_out/e62_skinny.txt 2>&1; echo "rc=$?" >> gpurun_out/e62_skinny.txt
