#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
python scripts/comb_probe.py 2 comb_one_role=1 > gpurun_out/comb.log 2>&1
python scripts/comb_probe.py 1 comb_one_role=1 >> gpurun_out/comb.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "combine or generate or chip or stream or blockoa or bench_path or dataset or slab" > gpurun_out/t.log 2>&1
