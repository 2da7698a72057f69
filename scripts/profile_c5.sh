#!/bin/bash
# ncu evidence for the config-5 headline (run on the GPU box after bench.py has
# exited 0 without ncu):
#  1. the launch list of one bench step (gpu__time_duration, cold / serialised):
#     each kernel's share of the step;
#  2. one --set full capture of each sweep kernel and of the combine/action
#     kernel (DRAM traffic, pipe utilisation, stalls).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 14000 --csv --log-file gpurun_out/r2_launches_c5.csv \
    python bench.py --steps 1 --warmup 3 --no-extra --no-e2e --no-cpu-baseline \
    > gpurun_out/r2_launches_c5.log 2>&1
echo "launches rc=$?" >> gpurun_out/r2_launches_c5.log
ncu --set full --import-source on --clock-control none \
    -k regex:"k_spmm64_ws|k_update64_ws|k_pupdate64_ws" --launch-skip 3 -c 3 \
    -o gpurun_out/r2_c5_sweeps python scripts/c5_phases.py 3 > gpurun_out/r2_c5_sweeps.log 2>&1
echo "sweeps rc=$?" >> gpurun_out/r2_c5_sweeps.log
ncu --set full --import-source on --clock-control none -k regex:"combine_action_kernel" -c 1 \
    -o gpurun_out/r2_c5_combine python scripts/comb_probe.py 5 500 > gpurun_out/r2_c5_combine.log 2>&1
echo "combine rc=$?" >> gpurun_out/r2_c5_combine.log
