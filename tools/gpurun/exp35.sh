mkdir -p gpurun_out
TBIK_TC_EPI=16 timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/e35_tests.log 2>&1
echo rc=$? >> gpurun_out/e35_tests.log
for e in 8 16 8 16; do TBIK_TC_EPI=$e timeout 300 python tools/ab_epi.py 1024 4096 2>&1 | grep -v Warn | sed "s/^/EPI=$e /"; done > gpurun_out/e35_epi.txt
