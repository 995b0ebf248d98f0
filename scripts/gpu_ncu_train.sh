#!/bin/bash
# ncu --set full of the C5 training kernels (one bench step)
out=${1:-gpurun_out/train}
mkdir -p $out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on \
  -k regex:"train_(fb|wgrad_tc)_kernel" -c 2 -o $out/prof_train -f \
  python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > $out/ncu_train.log 2>&1
tail -2 $out/ncu_train.log
