mkdir -p gpurun_out
TBIK_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/e30_n2.json 2> gpurun_out/e30_n2.err
echo rc=$? >> gpurun_out/e30_n2.err
