#!/bin/bash
# r02: default bench (N=1) + the N>1 code path on one GPU (TBIK_BENCH_SHARE_GPU=1: functional only).
mkdir -p gpurun_out
tag=${1:-r02_bench}
timeout 900 python bench.py > gpurun_out/${tag}_n1.json 2> gpurun_out/${tag}_n1.err; echo "rc=$?" >> gpurun_out/${tag}_n1.err
TBIK_BENCH_SHARE_GPU=1 timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-sweep --no-cpu > gpurun_out/${tag}_n2share.json 2> gpurun_out/${tag}_n2share.err; echo "rc=$?" >> gpurun_out/${tag}_n2share.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "rc=$?" >> gpurun_out/${tag}_ref.err
tail -3 gpurun_out/${tag}_*.err
