#!/bin/bash
# ncu --set full of the eta-sweep kernel (C4 shape, scripts/c4_time.py)
out=${1:-gpurun_out/eta}
mkdir -p $out
KREGEX=${KREGEX:-eta_sweep_pruned}
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -c 1 \
  -o $out/prof_eta -f python scripts/c4_time.py > $out/ncu_eta.log 2>&1
tail -3 $out/ncu_eta.log
