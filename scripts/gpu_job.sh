#!/bin/bash
# scratch job file for one gpurun call (the command of the latest A/B run)
cd $GRAFT_REPO_ROOT
python scripts/c5_loop_ab.py 3 > gpurun_out/ab3.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"k_ctl_alpha|k_ctl_update|k_update64_ws|k_spmm64_ws" -s 4 -c 4 -o gpurun_out/c5_ctl python scripts/c5_loop_ab.py 3 > gpurun_out/ncu_ctl.log 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-extra > gpurun_out/bench2.log 2>&1
