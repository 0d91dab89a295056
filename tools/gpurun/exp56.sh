mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_collective.py -q -x > gpurun_out/e56_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e56_pytest.log
S="4096 4096 28672 1024 4096 6144 1024 4096 128256 1024 4096 4096 4096 14336 4096"
timeout 200 python tools/ab_shape.py "pf4" $S > gpurun_out/e56.txt 2>&1
