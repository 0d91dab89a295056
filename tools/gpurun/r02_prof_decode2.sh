mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_skinny -s 5 -c 1 -o gpurun_out/r02s4_pd2 python tools/prof_decode.py 16 1792 4096 7 8 > gpurun_out/r02s4_pd2.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_active.avg,smsp__cycles_active.avg --clock-control none -k regex:"tc_skinny|nvjet" -c 12 --csv python tools/prof_decode.py 16 1792 4096 7 5 > gpurun_out/r02s4_pd2_t.csv 2>&1
tail -30 gpurun_out/r02s4_pd2_t.csv | cut -c1-250
