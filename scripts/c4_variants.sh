#!/bin/bash
# C4 eta-sweep timing per library variant (experiment builds, scripts/build_variant_file.sh)
for v in ${VARIANTS:-libdso_b200.so}; do
  echo "== $v"
  DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/$v timeout -s KILL 300 python scripts/c4_time.py 2>&1 | grep -v "prune=0"
done
