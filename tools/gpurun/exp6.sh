mkdir -p gpurun_out
timeout 300 python tools/e2e_chunks.py > gpurun_out/e6_chunks.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:ms_group|rmsnorm|finish' -s 3 -c 6 -o gpurun_out/e6_rowops python tools/rowops_bench.py > gpurun_out/e6_ncu.log 2>&1
timeout 900 python bench.py > gpurun_out/e6_bench.json 2> gpurun_out/e6_bench.err
