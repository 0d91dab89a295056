mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -k hostio -x -q > gpurun_out/e2_hostio.log 2>&1
timeout 600 python -m pytest tests/test_gpu_collective.py -x -q >> gpurun_out/e2_hostio.log 2>&1
timeout 900 python bench.py > gpurun_out/e2_bench.json 2> gpurun_out/e2_bench.err
