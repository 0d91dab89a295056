mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/e23_tests.log 2>&1
for d in 0 8; do TBIK_TC_DEBUG=$d timeout 300 python tools/ab_epi.py 1024 4096 2>&1 | grep -v Warn | sed "s/^/dbg=$d /"; done > gpurun_out/e23_dbg.txt
