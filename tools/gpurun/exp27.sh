mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/e27_tests.log 2>&1
for d in 1 0; do TBIK_TC_DEEP=$d timeout 300 python tools/ab_epi.py 1024 4096 2>&1 | grep -v Warn | grep "K=14336" | sed "s/^/deep=$d /"; done > gpurun_out/e27_deep.txt
for d in 1 0; do TBIK_TC_DEEP=$d timeout 300 python tools/ab_epi.py 1024 4096 2>&1 | grep -v Warn | grep "K=14336" | sed "s/^/deep=$d /"; done >> gpurun_out/e27_deep.txt
