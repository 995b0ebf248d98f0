set -u
OUT=gpurun_out/${1:-varc4}; mkdir -p $OUT
for v in ${VARIANTS}; do
  DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/$v timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > $OUT/$v.log 2>&1
done
