mkdir -p gpurun_out
timeout 1200 python tools/qwen_sweep.py > gpurun_out/e79_qwen.json 2> gpurun_out/e79_qwen.err; echo "rc=$?" >> gpurun_out/e79_qwen.err
timeout 600 python tools/fwd_profile.py > gpurun_out/e79_fwdprof.txt 2>&1; echo "rc=$?" >> gpurun_out/e79_fwdprof.txt
