mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_rowops.py -q -x > gpurun_out/e57_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e57_pytest.log
timeout 600 python tools/forward_bench.py --batch 4 --seq 256 > gpurun_out/e57_fwd.json 2>&1
timeout 300 python tools/fwd_profile.py 4 4 256 > gpurun_out/e57_fwdprof.txt 2>&1
