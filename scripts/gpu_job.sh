#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/b.log 2>&1
echo "bench rc=$?" >> gpurun_out/b.log
