mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -k "schedules" > gpurun_out/e45_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e45_pytest.log
S="4096 14336 4096 1024 14336 4096 2048 25600 5120"
timeout 120 python tools/ab_shape.py "narrow" $S > gpurun_out/e45.txt 2>&1
for st in 4 5 6; do for d in 0 1; do
  TBIK_TC_WIDE=1 TBIK_TC_WIDE_STAGES=$st TBIK_TC_DEBUG=$d timeout 120 python tools/ab_shape.py "wide st=$st dbg=$d" $S
done; done >> gpurun_out/e45.txt 2>&1
