mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_collective.py -q -x -k peer_group_processes > gpurun_out/e69_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e69_pytest.txt
