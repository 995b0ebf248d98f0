#!/bin/bash
# Round-2 evidence session: GPU tests, smoke, the default bench line (C3 headline +
# C2/C4/C5, e2e, cpu_baseline), reference arm, FMA-engine and dense-input lines,
# sanitizers (memcheck, racecheck, synccheck), launch lists, ncu --set full of the
# headline kernel and of the C4 / C5 kernels, per-role phase timing.
# Usage: gpurun --timeout 3600 -- bash scripts/gpu_r2.sh TAG
set -u
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
K="timeout -s KILL"
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nvidia-smi -q -d CLOCK >> $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu >> $OUT/nproc.txt 2>&1
( $K 1500 python -m pytest tests -q -m gpu --timeout 600 -rf -s > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log )
( $K 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log )
( $K 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.log 2>&1; echo "rc=$?" >> $OUT/bench.log )
( $K 600 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref.log 2>&1; echo "rc=$?" >> $OUT/bench_ref.log )
( $K 600 python bench.py --engine ffma --steps 10 --warmup 3 --no-cpu --no-e2e --no-stages --no-extra > $OUT/bench_ffma.log 2>&1; echo "rc=$?" >> $OUT/bench_ffma.log )
( $K 600 python bench.py --input dense --steps 10 --warmup 3 --no-cpu --no-e2e --no-stages --no-extra > $OUT/bench_dense.log 2>&1; echo "rc=$?" >> $OUT/bench_dense.log )
for tool in memcheck racecheck synccheck; do
  ( $K 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_run.py > $OUT/$tool.log 2>&1; echo "rc=$?" >> $OUT/$tool.log )
done
( $K 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --kernels 4194304 --no-e2e --no-cpu --no-stages --no-extra > $OUT/ncu_launch_bench.log 2>&1; echo "rc=$?" >> $OUT/ncu_launch_bench.log )
( $K 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv \
    python bench.py --config c5 --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1 )
( $K 900 ncu --set full --clock-control none --import-source on -k regex:"tc_kernel" -s 1 -c 1 \
    -o $OUT/prof_pipeline python bench.py --steps 1 --warmup 1 --kernels 2097152 --no-e2e --no-cpu --no-stages --no-extra > $OUT/ncu_full.log 2>&1; echo "rc=$?" >> $OUT/ncu_full.log )
( $K 900 ncu --set full --clock-control none --import-source on -k regex:ws_kernel -s 1 -c 1 \
    -o $OUT/prof_pipeline_ffma python bench.py --engine ffma --steps 1 --warmup 1 --kernels 2097152 --no-e2e --no-cpu --no-stages --no-extra > $OUT/ncu_full_ffma.log 2>&1; echo "rc=$?" >> $OUT/ncu_full_ffma.log )
( $K 600 ncu --set full --clock-control none -k regex:eta_sweep_pruned -s 1 -c 1 \
    -o $OUT/prof_eta python bench.py --config c4 --steps 1 --warmup 1 --kernels 1048576 --no-cpu > $OUT/ncu_eta.log 2>&1; echo "rc=$?" >> $OUT/ncu_eta.log )
( $K 600 ncu --set full --clock-control none -k regex:"train_fb|train_wgrad" -s 2 -c 2 \
    -o $OUT/prof_train python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > $OUT/ncu_train.log 2>&1; echo "rc=$?" >> $OUT/ncu_train.log )
( $K 300 python scripts/tc_phase.py > $OUT/tc_phase.txt 2>&1 )
ls -la $OUT
