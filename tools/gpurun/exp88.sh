mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_collective.py -q -x > gpurun_out/e88_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e88_pytest.txt
timeout 600 python tools/ab_debug.py --store > gpurun_out/e88_store.txt 2>&1; echo "rc=$?" >> gpurun_out/e88_store.txt
TBIK_TC_ACC4=0 timeout 300 python tools/ab_debug.py run 1792 4096 4096 > gpurun_out/e88_acc2.txt 2>&1
