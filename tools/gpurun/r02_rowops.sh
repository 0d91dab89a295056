#!/bin/bash
# r02: C5 row reductions (L2-flushed) incl. the fused lm_head + log-softmax, and the Llama forward.
mkdir -p gpurun_out
tag=${1:-r02_rowops}
timeout 400 python tools/rowops_bench.py > gpurun_out/${tag}_c5.json 2> gpurun_out/${tag}_c5.err
timeout 600 python tools/forward_bench.py --layers 32 --batch 4 --seq 256 > gpurun_out/${tag}_fwd.json 2> gpurun_out/${tag}_fwd.err
tail -c 1500 gpurun_out/${tag}_c5.json; echo; tail -c 1500 gpurun_out/${tag}_fwd.json; tail -3 gpurun_out/${tag}_c5.err gpurun_out/${tag}_fwd.err
