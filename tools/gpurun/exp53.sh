mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_model.py -q -x > gpurun_out/e53_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/e53_pytest.log
timeout 120 python tools/attn_bench.py > gpurun_out/e53_attn.txt 2>&1

timeout 600 python tools/forward_bench.py --batch 4 --seq 256 > gpurun_out/e53_fwd.json 2>&1
