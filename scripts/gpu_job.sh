#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/c5_phases.py 20 spmm_band=5 > gpurun_out/ph.log 2>&1
timeout 300 python scripts/c5_phases.py 20 spmm_band=5 >> gpurun_out/ph.log 2>&1
