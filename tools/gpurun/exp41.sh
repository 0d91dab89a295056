mkdir -p gpurun_out
for d in 0 1; do TBIK_TC_DEEP=$d timeout 300 python tools/tune_units.py 256 384 512 768 1024 2048 > gpurun_out/e41_deep$d.txt 2>&1; done
