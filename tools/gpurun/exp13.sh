mkdir -p gpurun_out
export CUDA_LAUNCH_BLOCKING=0
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/e13_tests.log 2>&1
echo "rc=$?" >> gpurun_out/e13_tests.log
timeout 600 python tools/tune_small.py 1 16 32 64 128 > gpurun_out/e13_small.txt 2>&1
