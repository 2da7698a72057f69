#!/bin/bash
# scratch job file for one gpurun call (edit, then: gpurun -- 'bash scripts/gpu_job.sh').
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 bash scripts/ab_lib.sh "PROBE_STREAMS=16 python scripts/batch_probe.py 2 16 3; PROBE_STREAMS=64 python scripts/batch_probe.py 1 64 3; BK_CG_PROFILE=1 PROBE_STREAMS=16 python scripts/batch_probe.py 2 16 3 2>&1 | grep profile | tail -n 1" > gpurun_out/ab.log 2>&1
for i in 1 2; do timeout 300 python -m pytest tests/test_gpu_stress.py tests/test_gpu_bench_path.py -q -x > gpurun_out/st$i.log 2>&1; echo "rc=$?" >> gpurun_out/st$i.log; done
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/t.log
