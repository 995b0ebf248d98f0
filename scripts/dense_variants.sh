#!/bin/bash
# dense-input C3 line per library variant (experiment builds, scripts/build_variant_file.sh)
for v in ${VARIANTS:-libdso_b200.so}; do
  echo "$v $(DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/$v timeout -s KILL 300 python bench.py --input dense --steps 10 --warmup 3 --no-cpu --no-e2e --no-stages --no-extra 2>&1 | grep -o '"ms_per_step": [0-9.]*')"
done
