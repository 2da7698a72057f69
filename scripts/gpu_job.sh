#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q -k "assemble or kat or mixed or csr or generate_chip" > gpurun_out/t.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-extra --no-e2e --no-cpu-baseline > gpurun_out/b.log 2>&1
