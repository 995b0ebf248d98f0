#!/bin/bash
# Iteration run: selected GPU test files (args after the tag), the headline bench
# line with stages (realistic mix, dense input), optional per-role phase timing.
# Usage: gpurun --timeout 1500 -- bash scripts/gpu_iter.sh TAG tests/test_x.py ...
set -u
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
( timeout -s KILL 420 python -m pytest "$@" -q -m gpu --timeout 120 -rf -x -s > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log )
( timeout -s KILL 300 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e --no-extra > $OUT/bench.log 2>&1; echo "rc=$?" >> $OUT/bench.log )
if [ "${PHASE:-0}" = "1" ]; then ( timeout -s KILL 200 python scripts/tc_phase.py > $OUT/tc_phase.txt 2>&1 ); fi
tail -3 $OUT/pytest.log
python - <<'PY' "$OUT/bench.log"
import json, sys
for l in open(sys.argv[1]):
    if l.startswith("{"):
        d = json.loads(l); r = d["roofline"]; st = d.get("stages") or {}
        rm = st.get("realistic_mix", {})
        print("C3 ms/step %.3f  value %.3e  frac %.3f  tensor %.3f | realistic tc %.2f ffma %.2f ms | dense %.2f" % (
            d["ms_per_step"], d["value"], r["frac"], r.get("tensor_view", {}).get("frac", 0),
            rm.get("tc_ms", 0), rm.get("ffma_ms", 0), st.get("pipeline_dense_input_ms", 0)))
PY
