#!/bin/bash
# One full ncu capture (source-level) of the tcgen05 pipeline kernel on the C3 bench stream.
# Usage: gpurun --timeout 900 -- bash scripts/gpu_ncu_tc.sh TAG [extra bench args]
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
( timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_kernel" -s 1 -c 1 \
    -o $OUT/prof_pipeline python bench.py --steps 1 --warmup 1 --kernels 2097152 --no-e2e --no-cpu --no-stages --no-extra "$@" > $OUT/ncu_full.log 2>&1; echo "rc=$?" >> $OUT/ncu_full.log )
tail -2 $OUT/ncu_full.log
