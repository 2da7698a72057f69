#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
python scripts/c5_loop_ab.py 3 > gpurun_out/ab3.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_spmm64_rs" -s 1 -c 1 -o gpurun_out/c5_rs4 python scripts/c5_loop_ab.py 3 > gpurun_out/ncu_rs.log 2>&1
