mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_gemm.py -x -q > gpurun_out/e42_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e42_pytest.log
for r in 1 2; do TBIK_RMS_ROWS=$r timeout 300 python tools/rowops_bench.py > gpurun_out/e42_rowops$r.json 2>&1; done
timeout 300 python tools/tune_units.py 256 512 1024 2048 4096 > gpurun_out/e42_units.txt 2>&1
timeout 600 python tools/forward_bench.py --batch 4 --seq 256 > gpurun_out/e42_fwd.json 2>&1
