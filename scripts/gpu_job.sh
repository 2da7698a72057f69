#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "large or c5 or fullsize or dd or graph or multikernel or slab or stress or duplicate or odd" > gpurun_out/t.log 2>&1
python scripts/c5_loop_ab.py > gpurun_out/ab.log 2>&1
python scripts/c5_loop_ab.py 3 > gpurun_out/ab3.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launch3.csv python scripts/c5_loop_ab.py 3 > gpurun_out/ncu3.log 2>&1
