mkdir -p gpurun_out
for mc in 0 1 0 1; do TBIK_TC_MC=$mc timeout 300 python tools/ab_epi.py 1024 4096 2>&1 | grep -v Warn | sed "s/^/mc=$mc /"; done > gpurun_out/e33_mc.txt
