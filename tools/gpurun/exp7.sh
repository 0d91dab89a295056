mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_rowops.py tests/test_gpu_model.py -x -q > gpurun_out/e7_tests.log 2>&1
timeout 300 python tools/rowops_bench.py > gpurun_out/e7_rowops.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:ms_group' -s 2 -c 1 -o gpurun_out/e7_msgroup python tools/rowops_bench.py > gpurun_out/e7_ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:finish|rmsnorm' -s 4 -c 2 -o gpurun_out/e7_fin python tools/rowops_bench.py > gpurun_out/e7_ncu2.log 2>&1
timeout 1200 python tools/qwen_sweep.py > gpurun_out/e7_qwen.json 2> gpurun_out/e7_qwen.err
