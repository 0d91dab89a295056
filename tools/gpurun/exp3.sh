mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_model.py -x -q > gpurun_out/e3_tests.log 2>&1
for d in 0 1 2 4; do TBIK_TC_DEBUG=$d timeout 300 python tools/ab_epi.py 1024 4096 2>&1 | grep -v Warn | sed "s/^/dbg=$d /"; done > gpurun_out/e3_dbg.txt
timeout 600 python tools/forward_bench.py --reps 3 > gpurun_out/e3_fwd.json 2>&1
