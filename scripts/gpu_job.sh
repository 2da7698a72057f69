#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 bash scripts/ab_lib.sh "python scripts/c5_phases.py 100; python scripts/c5_phases.py 100" > gpurun_out/ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "c5 or multikernel or s64 or slab or lookahead or graph_loop" > gpurun_out/t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t.log
