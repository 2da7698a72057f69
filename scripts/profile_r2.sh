#!/bin/bash
# Round-2 evidence for the config-5 headline, run on the GPU box:
#  1. the default bench line (no ncu);
#  2. the ncu launch list (gpu__time_duration, DRAM bytes; cold / serialised) of
#     one bench step's first ~280 solve iterations (warm-up launches skipped);
#  3. one --set full capture of each S = 64 sweep and of the C5 / C2
#     combine-action kernels (the same commands ran clean first).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python bench.py > gpurun_out/r2_bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/r2_bench.log
CMD="python bench.py --steps 1 --warmup 3 --no-extra --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/r2_launch_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -s 17400 -c 2000 --csv --log-file gpurun_out/r2_launches_c5.csv $CMD > gpurun_out/r2_launches.log 2>&1
echo "launches rc=$?" >> gpurun_out/r2_launches.log
python scripts/c5_loop_ab.py 3 > gpurun_out/r2_sweeps_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none \
    -k regex:"k_spmm64_rs|k_update64_ws|k_pupdate64_ws|k_ctl_alpha" -s 4 -c 4 \
    -o gpurun_out/r2_c5_sweeps python scripts/c5_loop_ab.py 3 > gpurun_out/r2_c5_sweeps.log 2>&1
echo "sweeps rc=$?" >> gpurun_out/r2_c5_sweeps.log
python scripts/comb_probe.py 5 500 > gpurun_out/r2_comb_plain.log 2>&1 && \
python scripts/comb_probe.py 2 >> gpurun_out/r2_comb_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"combine_action" -c 1 \
    -o gpurun_out/r2_c5_combine python scripts/comb_probe.py 5 500 > gpurun_out/r2_c5_combine.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:"combine_action" -c 1 \
    -o gpurun_out/r2_c2_combine python scripts/comb_probe.py 2 > gpurun_out/r2_c2_combine.log 2>&1
echo "combine rc=$?" >> gpurun_out/r2_c5_combine.log
