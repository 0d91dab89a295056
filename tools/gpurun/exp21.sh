mkdir -p gpurun_out
for pf in 0 4 8 16 32; do TBIK_TC_PF=$pf timeout 300 python tools/ab_epi.py 1024 4096 2>&1 | grep -v Warn | sed "s/^/pf=$pf /"; done > gpurun_out/e21_pf.txt
