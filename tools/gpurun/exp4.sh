mkdir -p gpurun_out
for st in 8 6; do for d in 0 8 10 1; do TBIK_TC_STAGES=$st TBIK_TC_DEBUG=$d timeout 300 python tools/ab_epi.py 4096 2>&1 | grep -v Warn | sed "s/^/st=$st dbg=$d /"; done; done > gpurun_out/e4_dbg.txt
