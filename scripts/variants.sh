# bench the C3 pipeline with alternative library builds (role placement / sweep split)
set -u
OUT=gpurun_out/${1:-var}; mkdir -p $OUT
for v in libdso_b200.so libdso_b200_v1_32.so libdso_b200_v0_64.so libdso_b200_v0_32.so; do
  DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/$v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-stages > $OUT/$v.log 2>&1
  DSO_B200_LIB=$PWD/paper_2407_13096_b200/lib/$v timeout 300 python -m pytest tests/test_gpu_pipeline.py -q -x > $OUT/$v.pytest 2>&1
done
