mkdir -p gpurun_out
timeout 600 python tools/ab_debug.py --store > gpurun_out/e87_store.txt 2>&1; echo "rc=$?" >> gpurun_out/e87_store.txt
