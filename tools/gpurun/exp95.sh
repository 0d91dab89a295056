mkdir -p gpurun_out
timeout 1200 python tools/qwen_sweep.py > gpurun_out/e95_qwen.json 2> gpurun_out/e95_qwen.err; echo "rc=$?" >> gpurun_out/e95_qwen.err
