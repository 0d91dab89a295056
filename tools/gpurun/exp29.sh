mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/e29_tests.log 2>&1
echo rc=$? >> gpurun_out/e29_tests.log
for d in 1 0; do TBIK_TC_DEEP=$d timeout 600 python tools/tune_small.py 1 16 64 128 256 2>&1 | grep -v Warn | sed "s/^/deep=$d /"; done > gpurun_out/e29_small.txt
timeout 300 python tools/ab_epi.py 1024 4096 > gpurun_out/e29_ab.txt 2>&1
