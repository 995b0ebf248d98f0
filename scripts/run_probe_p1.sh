set -u
OUT=gpurun_out/p1; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/probes/lds_probe scripts/probes/lds_probe.cu
ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__inst_executed_op_shared_ld.sum --csv scripts/probes/lds_probe > $OUT/lds_probe.csv 2>&1
timeout 900 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_mlp.py tests/test_gpu_cpp.py -q -x > $OUT/pytest.log 2>&1; echo rc=$? >> $OUT/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/bench.log 2>&1
timeout 600 python bench.py --config c2 --steps 20 --warmup 3 --no-cpu --no-e2e > $OUT/bench_c2.log 2>&1
timeout 600 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active -k regex:ws_kernel -s 1 -c 1 python bench.py --steps 1 --warmup 1 --kernels 2097152 --no-e2e --no-cpu --no-stages > $OUT/ncu_ws.log 2>&1
