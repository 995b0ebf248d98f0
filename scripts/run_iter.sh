# iteration loop on the GPU box: targeted tests, C3/C2/C4 bench lines, phase timing
set -u
OUT=gpurun_out/${1:-it}; mkdir -p $OUT
timeout 900 python -m pytest ${TESTS:-tests/test_gpu_sweep.py tests/test_gpu_pipeline.py} -q -x > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/bench.log 2>&1
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu --no-e2e > $OUT/bench_c2.log 2>&1
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu --no-e2e > $OUT/bench_c4.log 2>&1
timeout 300 python scripts/phase_timing.py > $OUT/phase.txt 2>&1
