mkdir -p gpurun_out
timeout 300 python tools/skinny_check.py > gpurun_out/e65_skinny.txt 2>&1; echo "rc=$?" >> gpurun_out/e65_skinny.txt
timeout 300 python tools/decode_bench.py > gpurun_out/e65_decode.txt 2>&1; echo "rc=$?" >> gpurun_out/e65_decode.txt
