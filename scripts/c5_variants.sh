#!/bin/bash
# C5 gradient timing per library variant (experiment builds, scripts/build_variant_file.sh)
for v in ${VARIANTS:-libdso_b200.so}; do
  echo "$v $(DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/$v timeout -s KILL 200 python scripts/c5_probe.py 2>&1 | grep 'train_tc=1')"
done
