#!/bin/bash
# combine + action alone on C2, C3 and C5 (500 samples) operators
cd "$(dirname "$0")/.."
for c in 2 3; do python scripts/comb_probe.py $c; done
python scripts/comb_probe.py 5 500
