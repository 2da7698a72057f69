#!/bin/bash
# A/B: run a command with the current library and with scripts/ab/libblockoa_b200_before.so
cd "$(dirname "$0")/.."
echo "== after"; bash -c "$*"
cp paper_2510_23221_b200/libblockoa_b200.so /tmp/lib_after.so
cp scripts/ab/libblockoa_b200_before.so paper_2510_23221_b200/libblockoa_b200.so
echo "== before"; bash -c "$*"
cp /tmp/lib_after.so paper_2510_23221_b200/libblockoa_b200.so
