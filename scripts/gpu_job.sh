#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_stress.py -q -x > gpurun_out/st$i.log 2>&1; echo "rc=$?" >> gpurun_out/st$i.log; done
timeout 300 python -m pytest tests/test_gpu_bench_path.py tests/test_gpu_fullsize.py -q -x > gpurun_out/t.log 2>&1; echo "rc=$?" >> gpurun_out/t.log
