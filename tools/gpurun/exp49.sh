mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -k "schedules or wide" > gpurun_out/e49_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e49_pytest.log
S="4096 14336 4096 1024 14336 4096 2048 25600 5120 4096 4096 28672"
timeout 120 python tools/ab_shape.py "narrow" $S > gpurun_out/e49.txt 2>&1
for st in 5 6; do for d in 0 4; do
  TBIK_TC_WIDE=1 TBIK_TC_WIDE_STAGES=$st TBIK_TC_DEBUG=$d timeout 120 python tools/ab_shape.py "wide st=$st dbg=$d" $S
done; done >> gpurun_out/e49.txt 2>&1
TBIK_TC_WIDE=1 TBIK_TC_WIDE_SPLIT=0 timeout 120 python tools/ab_shape.py "wide nosplit" $S >> gpurun_out/e49.txt 2>&1
