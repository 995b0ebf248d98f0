#!/bin/bash
# quick, hang-safe check of the tc engine: smoke, short bench, trace, focused tests
OUT=gpurun_out/${1:-tcq}; mkdir -p $OUT
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "rc=$?" >> $OUT/smoke.log
timeout 120 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-stages --no-extra > $OUT/bench.log 2>&1; echo "rc=$?" >> $OUT/bench.log
timeout 120 python scripts/tc_trace.py > $OUT/trace.txt 2>&1
timeout 600 python -m pytest ${TESTS:-tests/test_gpu_pipeline.py tests/test_gpu_tc.py tests/test_gpu_mlp.py} -q -x -m gpu --timeout 120 > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
