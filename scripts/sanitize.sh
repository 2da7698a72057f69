#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_cases.py
# (every block-CG instantiation, combine/action, the stream pipeline and
# generate_blockoa on reduced shapes). Logs to gpurun_out/sanitizer_<tool>.log.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
    timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_cases.py \
        > gpurun_out/sanitizer_$tool.log 2>&1
    echo "tool=$tool rc=$?" >> gpurun_out/sanitizer_$tool.log
done
