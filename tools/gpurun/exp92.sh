mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_collective.py -q -x > gpurun_out/e92_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e92_pytest.txt
