#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 bash scripts/ab_lib.sh "python scripts/comb_probe.py 5 32; python scripts/comb_probe.py 5 500; python scripts/comb_probe.py 3 200; python scripts/comb_probe.py 3; python scripts/comb_probe.py 4 8" > gpurun_out/ab.log 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "combine or generate_chip or slab_local or blockoa or stream" > gpurun_out/t.log 2>&1; echo "rc=$?" >> gpurun_out/t.log
