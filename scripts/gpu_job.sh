#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do timeout 600 python -m pytest tests/test_gpu_stress.py -q -k "batched_solve_and_combine_repeatable" > gpurun_out/st$i.log 2>&1; echo "rc=$?" >> gpurun_out/st$i.log; done
timeout 1500 python -m pytest tests -m gpu -q -x --durations=5 > gpurun_out/t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t.log
