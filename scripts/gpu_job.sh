#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 bash scripts/ab_lib.sh "python scripts/comb_probe.py 2 comb_one_role=1; python scripts/comb_probe.py 1 comb_one_role=1; python scripts/comb_probe.py 2 comb_one_role=1" > gpurun_out/ab.log 2>&1
