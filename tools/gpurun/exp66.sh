mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "skinny or schedules or tree_over or tp_invariance or batch" > gpurun_out/e66_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e66_pytest.txt
timeout 300 python tools/decode_bench.py 1 16 32 64 128 > gpurun_out/e66_decode.txt 2>&1; echo "rc=$?" >> gpurun_out/e66_decode.txt
