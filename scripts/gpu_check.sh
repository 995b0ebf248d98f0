#!/bin/bash
# One gpurun session: GPU tests, smoke, short bench, launch list + one full ncu capture.
# Usage (from the build container):
#   gpurun --timeout 2400 -- bash scripts/gpu_check.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nvidia-smi -q -d CLOCK >> $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu >> $OUT/nproc.txt 2>&1
( timeout 1200 python -m pytest tests -q -m gpu --timeout 600 -rf > $OUT/pytest_gpu.log 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.log ) 
( timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log )
( timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python scripts/sanitize_run.py > $OUT/memcheck.log 2>&1; echo "rc=$?" >> $OUT/memcheck.log )
( timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench.log 2>&1; echo "rc=$?" >> $OUT/bench.log )
( timeout 600 python bench.py --config c5 --steps 10 --warmup 3 > $OUT/bench_c5.log 2>&1; echo "rc=$?" >> $OUT/bench_c5.log )
( timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu > $OUT/bench_c2.log 2>&1; echo "rc=$?" >> $OUT/bench_c2.log )
( timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu > $OUT/bench_c4.log 2>&1; echo "rc=$?" >> $OUT/bench_c4.log )
( timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 2 --warmup 1 --kernels 4194304 --no-e2e --no-cpu > $OUT/ncu_launch_bench.log 2>&1; echo "rc=$?" >> $OUT/ncu_launch_bench.log )
( timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_kernel|ws_kernel" -s 1 -c 1 \
    -o $OUT/prof_pipeline python bench.py --steps 1 --warmup 1 --kernels 2097152 --no-e2e --no-cpu --no-stages > $OUT/ncu_full.log 2>&1; echo "rc=$?" >> $OUT/ncu_full.log )
( timeout 900 ncu --set full --clock-control none --import-source on -k regex:ws_kernel -s 1 -c 1 \
    -o $OUT/prof_pipeline_ffma python bench.py --engine ffma --steps 1 --warmup 1 --kernels 2097152 --no-e2e --no-cpu --no-stages > $OUT/ncu_full_ffma.log 2>&1; echo "rc=$?" >> $OUT/ncu_full_ffma.log )
( timeout 600 python bench.py --engine ffma --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/bench_ffma.log 2>&1; echo "rc=$?" >> $OUT/bench_ffma.log )
( timeout 600 python bench.py --input dense --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/bench_dense.log 2>&1; echo "rc=$?" >> $OUT/bench_dense.log )
( timeout 300 python scripts/tc_phase.py > $OUT/tc_phase.txt 2>&1 )
( timeout 600 ncu --set full --clock-control none --import-source on -k regex:eta_sweep_fast -s 1 -c 1 \
    -o $OUT/prof_eta python bench.py --config c4 --steps 1 --warmup 1 --kernels 1048576 --no-cpu > $OUT/ncu_eta.log 2>&1; echo "rc=$?" >> $OUT/ncu_eta.log )
( timeout 600 ncu --set full --clock-control none --import-source on -k regex:"train_fb|train_wgrad" -s 2 -c 2 \
    -o $OUT/prof_train python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > $OUT/ncu_train.log 2>&1; echo "rc=$?" >> $OUT/ncu_train.log )
( timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv \
    python bench.py --config c5 --steps 2 --warmup 1 --no-cpu > /dev/null 2>&1 )
( timeout 300 python scripts/phase_timing.py > $OUT/phase_timing.txt 2>&1 )
ls -la $OUT
