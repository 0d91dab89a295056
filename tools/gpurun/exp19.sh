mkdir -p gpurun_out
timeout 120 python tools/attn_bench.py > gpurun_out/e19_attn.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_model.py -x -q >> gpurun_out/e19_attn.txt 2>&1
cp tools/ab/libtbik_old.so paper_2511_17826_b200/libtbik_b200.so
echo "old:" >> gpurun_out/e19_attn.txt
timeout 120 python tools/attn_bench.py >> gpurun_out/e19_attn.txt 2>&1
