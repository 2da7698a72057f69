#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
bash scripts/ab_lib.sh python scripts/small_solve_bench.py > gpurun_out/ss.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1
