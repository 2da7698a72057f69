#!/bin/bash
# scratch job file for one gpurun call (edit, then: gpurun -- 'bash scripts/gpu_job.sh').
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-extra --no-e2e --no-cpu-baseline --no-dd-leg > gpurun_out/b.log 2>&1
echo "bench rc=$?" >> gpurun_out/b.log
