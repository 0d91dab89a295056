mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/e94_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e94_pytest.txt
timeout 600 python tools/midm_sweep.py > gpurun_out/e94_midm.txt 2>&1; echo "rc=$?" >> gpurun_out/e94_midm.txt
