mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x -k "wide" > gpurun_out/e51_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e51_pytest.log
S="4096 14336 4096 2048 25600 5120"
for kb in 1 2 4; do for d in 0 1 4; do
  TBIK_TC_WIDE=1 TBIK_TC_WIDE_STAGES=6 TBIK_TC_WIDE_KB=$kb TBIK_TC_DEBUG=$d timeout 120 python tools/ab_shape.py "wide kb=$kb dbg=$d" $S
done; done > gpurun_out/e51.txt 2>&1
