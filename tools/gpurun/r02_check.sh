#!/bin/bash
# r02: full GPU suite + smoke + a short bench (no sweep/forward) -- the regression check after a change.
mkdir -p gpurun_out
tag=${1:-r02_check}
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/${tag}.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
timeout 600 python bench.py --no-sweep --no-forward --no-cpu > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err
tail -15 gpurun_out/${tag}.log; tail -2 gpurun_out/${tag}_smoke.log; head -c 300 gpurun_out/${tag}_bench.json
