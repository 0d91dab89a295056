mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x > gpurun_out/e59_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e59_pytest.log
timeout 300 python tools/fma_bench.py > gpurun_out/e59_fma.txt 2>&1
