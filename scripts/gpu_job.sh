#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "64_chips or measure_fp64 or generate_batch" > gpurun_out/t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t.log
timeout 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/b_c1.log 2>&1; echo "rc=$?" >> gpurun_out/b_c1.log
