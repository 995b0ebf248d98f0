# bench the C3 pipeline (headline only) with alternative library builds (experiments)
set -u
OUT=gpurun_out/${1:-var}; mkdir -p $OUT
for v in ${VARIANTS:-libdso_b200.so}; do
  DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-stages --no-extra > $OUT/$v.log 2>&1
  echo "$v $(grep -o '"ms_per_step": [0-9.]*' $OUT/$v.log | head -1)" | tee -a $OUT/summary.txt
done
