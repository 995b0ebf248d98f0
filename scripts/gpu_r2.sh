#!/bin/bash
# Round-2 GPU session: full GPU tests, smoke, the default bench line (headline +
# C2/C4/C5), sanitizers (memcheck, racecheck, synccheck), launch list, one full ncu
# capture of the headline kernel.  Usage: gpurun --timeout 3000 -- bash scripts/gpu_r2.sh TAG [quick]
set -u
TAG=${1:-r2}
MODE=${2:-full}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
( timeout 1500 python -m pytest tests -q -m gpu --timeout 900 -rf -s > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log )
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log )
( timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.log 2>&1; echo "rc=$?" >> $OUT/bench.log )
( timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.log 2>&1; echo "rc=$?" >> $OUT/bench_ref.log )
if [ "$MODE" = "full" ]; then
for tool in memcheck racecheck synccheck; do
  ( timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > $OUT/$tool.log 2>&1; echo "rc=$?" >> $OUT/$tool.log )
done
( timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-stages --no-extra > $OUT/ncu_launch_bench.log 2>&1; echo "rc=$?" >> $OUT/ncu_launch_bench.log )
( timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_kernel" -s 1 -c 1 \
    -o $OUT/prof_pipeline python bench.py --steps 1 --warmup 1 --kernels 2097152 --no-e2e --no-cpu --no-stages --no-extra > $OUT/ncu_full.log 2>&1; echo "rc=$?" >> $OUT/ncu_full.log )
fi
ls -la $OUT
