mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/e74_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e74_pytest.txt
timeout 600 python tools/ab_debug.py > gpurun_out/e74_ab.txt 2>&1; echo "rc=$?" >> gpurun_out/e74_ab.txt
