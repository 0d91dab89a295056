#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_model.py -q -x -m gpu > gpurun_out/r02_rq_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/r02_rq_tests.log
tail -n 2 gpurun_out/r02_rq_tests.log
for i in 1 2; do timeout 900 python tools/forward_bench.py > gpurun_out/r02_rq_fwd_$i.txt 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r02_rq_fwd_$i.txt').read().strip().splitlines()[-1]); print(d['tbik_tokens_per_s'], d['tbik_graph_tokens_per_s'], d['noninvariant_tokens_per_s'], d.get('noninvariant_graph_tokens_per_s'), d['logits_bit_identical'], d['graph_bit_identical_to_eager'])"; done
