#!/bin/bash
cd $GRAFT_REPO_ROOT
python scripts/comb_probe.py 2 > gpurun_out/comb2.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"combine_action_pl_ws" -s 1 -c 1 -o gpurun_out/comb2ws3 python scripts/comb_probe.py 2 > gpurun_out/ncu_comb2.log 2>&1
