#!/bin/bash
# Iteration run + memcheck of the sanitize script.  Usage: gpu_iter2.sh TAG tests...
set -u
TAG=$1
bash scripts/gpu_iter.sh "$@"
OUT=gpurun_out/$TAG
( timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_run.py > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log )
tail -3 $OUT/memcheck.log
