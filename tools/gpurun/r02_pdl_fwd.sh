#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/r02_pdlf_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r02_pdlf_pytest.log
tail -n 2 gpurun_out/r02_pdlf_pytest.log
for i in 1 2; do timeout 900 python tools/forward_bench.py > gpurun_out/r02_pdlf_fwd_$i.txt 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r02_pdlf_fwd_$i.txt').read().strip().splitlines()[-1]); print(d['tbik_tokens_per_s'], d['tbik_graph_tokens_per_s'], d['noninvariant_tokens_per_s'], d.get('noninvariant_graph_tokens_per_s'), d['logits_bit_identical'])"; done
