#!/bin/bash
# C5 combine/action kernel: plain timing, then one --set full capture with source
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/comb_probe.py 5 500 > gpurun_out/comb_plain.log 2>&1
echo "plain rc=$?" >> gpurun_out/comb_plain.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"combine_action" -c 1 \
    -o gpurun_out/c5_combine python scripts/comb_probe.py 5 500 > gpurun_out/c5_combine_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/c5_combine_ncu.log
