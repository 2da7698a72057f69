#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
BK_COMB_PROFILE=1 python scripts/comb_probe.py 5 500 > gpurun_out/ab.log 2>&1
BK_COMB_PROFILE=1 python scripts/comb_probe.py 3 >> gpurun_out/ab.log 2>&1
