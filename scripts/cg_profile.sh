#!/bin/bash
# per-phase timing of the block CG kernel (BK_CG_PROFILE prints to stderr)
export BK_CG_PROFILE=1
python scripts/prof_chip.py 2 2
python scripts/prof_chip.py 1 2
python scripts/prof_chip.py 3 1
