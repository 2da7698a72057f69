#!/bin/bash
# one gpurun call: full GPU suite, smoke, and the default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/b.log 2>&1
echo "bench rc=$?" >> gpurun_out/b.log
