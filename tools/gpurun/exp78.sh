mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_model.py -q -x > gpurun_out/e78_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e78_pytest.txt
timeout 600 python tools/rowops_bench.py > gpurun_out/e78_rowops.txt 2>&1; echo "rc=$?" >> gpurun_out/e78_rowops.txt
