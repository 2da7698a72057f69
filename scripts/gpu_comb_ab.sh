#!/bin/bash
# combine/action A/B on one box: current library (units and m-tile forms) vs
# scripts/ab/libblockoa_b200_before.so
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
P="python scripts/comb_probe.py"
bash scripts/ab_lib.sh "$P 5 500 comb_mtile=1; $P 3; $P 5 500" > gpurun_out/comb_ab.log 2>&1
echo "ab rc=$?" >> gpurun_out/comb_ab.log
