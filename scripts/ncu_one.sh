# one ncu --set full capture of the fused kernel (2M kernels) + its source page
set -u
OUT=gpurun_out/${1:-ncu}; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-ws_kernel} -s ${SKIP:-1} -c 1 \
    -o $OUT/prof python bench.py ${BENCH_ARGS:---steps 1 --warmup 1 --kernels 2097152 --no-e2e --no-cpu --no-stages} > $OUT/ncu.log 2>&1
echo rc=$? >> $OUT/ncu.log
