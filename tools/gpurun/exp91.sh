mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_model.py -q -x > gpurun_out/e91_pytest.txt 2>&1; echo "rc=$?" >> gpurun_out/e91_pytest.txt
timeout 1200 python tools/qwen_sweep.py > gpurun_out/e91_qwen.json 2> gpurun_out/e91_qwen.err; echo "rc=$?" >> gpurun_out/e91_qwen.err
