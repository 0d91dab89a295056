#!/bin/bash
mkdir -p gpurun_out
for cfg in "0 4 256" "1 4 256" "0 1 2048" "1 1 2048" "0 8 512" "1 8 512"; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"attn_mma|attn_tc5" -c 3 --csv python tools/prof_attn.py $cfg > gpurun_out/tc5p.csv 2>&1
  python - "$cfg" <<'PY'
import csv, sys
rows=[r for r in csv.reader(open('gpurun_out/tc5p.csv')) if len(r)>10]
h=rows[0]; vi=h.index("Metric Value")
print(sys.argv[1], [r[vi] for r in rows[1:]])
PY
done
