mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_collective.py -q -x > gpurun_out/e90_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e90_pytest.txt
for K in 14336 7168 3584 1792; do
  for n in 2 9; do
    echo "K=$K nacc_cap=$n $(TBIK_TC_NACC=$n timeout 300 python tools/ab_debug.py run $K 4096 4096)" >> gpurun_out/e90_nacc.txt
  done
done
for K in 4096; do for M in 1024 2048; do
  for n in 2 9; do
    echo "K=$K M=$M nacc_cap=$n $(TBIK_TC_NACC=$n timeout 300 python tools/ab_debug.py run $K 4096 $M)" >> gpurun_out/e90_nacc.txt
  done
done; done
