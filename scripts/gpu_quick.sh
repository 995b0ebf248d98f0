#!/bin/bash
# Quick GPU iteration: selected GPU test files (args) + headline bench line.
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
( timeout 1200 python -m pytest "$@" -q -m gpu --timeout 600 -rf -x -s > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log )
( timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-stages --no-e2e --no-extra > $OUT/bench.log 2>&1; echo "rc=$?" >> $OUT/bench.log )
tail -3 $OUT/pytest.log; grep -o '"value": [0-9.e+]*, "unit": "(kernel, freq-pair) evals/s", "n_gpus": [0-9]*, "steps": [0-9]*, "warmup": [0-9]*, "ms_per_step": [0-9.]*' $OUT/bench.log
