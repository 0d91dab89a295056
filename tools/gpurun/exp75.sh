mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/e75_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e75_pytest.txt
timeout 600 python tools/ab_debug.py > gpurun_out/e75_ab.txt 2>&1; echo "rc=$?" >> gpurun_out/e75_ab.txt
timeout 600 python tools/midm_sweep.py > gpurun_out/e75_midm.txt 2>&1; echo "rc=$?" >> gpurun_out/e75_midm.txt
