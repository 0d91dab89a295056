mkdir -p gpurun_out
timeout 300 python tools/decode_bench.py 16 64 > gpurun_out/e80_decode.txt 2>&1; echo "rc=$?" >> gpurun_out/e80_decode.txt
timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x -k skinny > gpurun_out/e80_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e80_pytest.txt
