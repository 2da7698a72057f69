#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/c5_phases.py 20 update_teams=1 > gpurun_out/ph.log 2>&1
timeout 300 python scripts/c5_phases.py 20 update_teams=1 >> gpurun_out/ph.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "large or c5 or fullsize or graph or multikernel or slab or stress" > gpurun_out/t.log 2>&1
