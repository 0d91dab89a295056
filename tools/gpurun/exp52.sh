mkdir -p gpurun_out
timeout 300 python tools/fwd_profile.py 4 4 256 > gpurun_out/e52_fwdprof.txt 2>&1
