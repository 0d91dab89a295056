mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e14_tests.log 2>&1
echo "rc=$?" >> gpurun_out/e14_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e14_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/e14_bench.json 2> gpurun_out/e14_bench.err
timeout 900 python tools/forward_bench.py --batch 1 --seq 16 --reps 5 --tps 1,8 > gpurun_out/e14_fwd_small.json 2>&1
