#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
python scripts/ctl_solve_bench.py > gpurun_out/ctl_solve.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k "large or c5 or fullsize or dd or graph or multikernel or slab or stress" > gpurun_out/t.log 2>&1
python scripts/c5_loop_ab.py > gpurun_out/ab.log 2>&1
python scripts/c5_phases.py 20 > gpurun_out/ph.log 2>&1
