#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/solve_ab.py 3 12 no_pencil=1 > gpurun_out/ab.log 2>&1
BK_CG_PROFILE=1 timeout 300 python scripts/solve_ab.py 3 8 >> gpurun_out/ab.log 2>&1
