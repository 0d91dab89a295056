mkdir -p gpurun_out
./tools/micro/tmem_ld_bw > gpurun_out/e1_tmem.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_collective.py -x -q > gpurun_out/e1_coll.log 2>&1
for d in 0 1 2 4; do TBIK_TC_DEBUG=$d timeout 300 python tools/ab_epi.py 4096 2>&1 | grep -v Warn | sed "s/^/dbg=$d /"; done > gpurun_out/e1_dbg.txt
timeout 300 python tools/ab_wide.py 1024 4096 > gpurun_out/e1_wide.txt 2>&1
