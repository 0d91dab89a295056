mkdir -p gpurun_out
for gm in 8 1 2 4 16 32; do TBIK_TC_GROUP_M=$gm timeout 300 python tools/ab_epi.py 4096 2>&1 | grep -v Warn | head -2 | sed "s/^/gm=$gm /"; done > gpurun_out/e22_gm.txt
