mkdir -p gpurun_out
timeout 600 python tools/skinny_units.py > gpurun_out/e96_units.txt 2>&1; echo "rc=$?" >> gpurun_out/e96_units.txt
