#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python scripts/d2h_bw.py > gpurun_out/d2h.log 2>&1
bash scripts/ab_lib.sh "python scripts/c5_stream_probe.py 3" > gpurun_out/ab.log 2>&1
