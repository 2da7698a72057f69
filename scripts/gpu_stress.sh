#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do timeout 600 python -m pytest tests/test_gpu_stress.py -q -k "repeatable" > gpurun_out/st$i.log 2>&1; echo "rc=$?" >> gpurun_out/st$i.log; done
