mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_model.py tests/test_gpu_gemm.py -x -q > gpurun_out/e38_tests.log 2>&1
echo rc=$? >> gpurun_out/e38_tests.log
timeout 900 python tools/forward_bench.py --reps 3 --tps 1,8 > gpurun_out/e38_fwd.json 2>&1
