mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rowops.py -q -x > gpurun_out/e58_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e58_pytest.log
timeout 300 python tools/rowops_bench.py > gpurun_out/e58_rowops.json 2>&1
