mkdir -p gpurun_out
timeout 120 tools/micro/tma_stream > gpurun_out/e64_tma_stream.txt 2>&1; echo rc=$? >> gpurun_out/e64_tma_stream.txt
