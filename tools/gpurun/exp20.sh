mkdir -p gpurun_out
timeout 120 python tools/attn_bench.py > gpurun_out/e20_attn.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_model.py -x -q >> gpurun_out/e20_attn.txt 2>&1
