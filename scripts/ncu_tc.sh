set -u
OUT=gpurun_out/${1:-ncu_tc1}; mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_kernel -s 1 -c 1 \
    -o $OUT/prof python bench.py --steps 1 --warmup 1 --kernels 1048576 --no-e2e --no-cpu --no-stages > $OUT/ncu.log 2>&1
echo rc=$? >> $OUT/ncu.log
ncu -i $OUT/prof.ncu-rep --page source --csv --print-source cuda,sass > $OUT/src.csv 2>/dev/null
python scripts/ncu_toplines.py $OUT/src.csv "" 60 > $OUT/toplines.txt
