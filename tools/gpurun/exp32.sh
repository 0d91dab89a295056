mkdir -p gpurun_out
TBIK_TC_MC=1 timeout 300 python tools/ab_epi.py 4096 > gpurun_out/e32_mc.txt 2>&1
echo "rc=$?" >> gpurun_out/e32_mc.txt
TBIK_TC_MC=1 timeout 600 python -m pytest tests/test_gpu_gemm.py -x -q > gpurun_out/e32_tests.log 2>&1
echo "rc=$?" >> gpurun_out/e32_tests.log
for mc in 0 1 0 1; do TBIK_TC_MC=$mc timeout 300 python tools/ab_epi.py 1024 4096 2>&1 | grep -v Warn | sed "s/^/mc=$mc /"; done >> gpurun_out/e32_mc.txt
