#!/bin/bash
# scratch job file for one gpurun call (edit, then: gpurun -- 'bash scripts/gpu_job.sh').
# Typical A/B: build the old library into scripts/ab/libblockoa_b200_before.so and run
#   bash scripts/ab_lib.sh "python scripts/c5_phases.py 100"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3 4 5 6; do timeout 300 python -m pytest tests/test_gpu_stress.py tests/test_gpu_bench_path.py -q -x > gpurun_out/st$i.log 2>&1; echo "rc=$?" >> gpurun_out/st$i.log; done
for i in 1 2; do timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/full$i.log 2>&1; echo "pytest rc=$?" >> gpurun_out/full$i.log; done
