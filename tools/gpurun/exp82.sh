mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k "skinny or schedules" > gpurun_out/e82_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e82_pytest.txt
timeout 300 python tools/decode_bench.py 16 > gpurun_out/e82_decode.txt 2>&1; echo "rc=$?" >> gpurun_out/e82_decode.txt
