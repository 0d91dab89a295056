#!/bin/bash
# r02: the whole GPU test suite + smoke (what the driver runs at round end).
mkdir -p gpurun_out
tag=${1:-r02_suite}
timeout 2400 python -m pytest tests/ -q -m gpu -x -p no:cacheprovider > gpurun_out/${tag}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${tag}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/${tag}_smoke.log
tail -n 3 gpurun_out/${tag}_pytest.log gpurun_out/${tag}_smoke.log
