#!/bin/bash
# scratch job file for one gpurun call (edit, then: gpurun -- 'bash scripts/gpu_job.sh').
# Typical A/B: build the old library into scripts/ab/libblockoa_b200_before.so and run
#   bash scripts/ab_lib.sh "python scripts/c5_phases.py 100"
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t.log
