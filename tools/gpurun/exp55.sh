mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_model.py -q -x -k "rope" > gpurun_out/e55_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e55_pytest.log
S="4096 4096 28672 1024 4096 6144 1024 4096 128256"
for d in 0 1 2 4 8 16; do
  TBIK_TC_DEBUG=$d timeout 120 python tools/ab_shape.py "narrow dbg=$d" $S
done > gpurun_out/e55.txt 2>&1
