# A/B of the two predictor engines on the bench configs (GPU box)
set -u
OUT=gpurun_out/${1:-ab}; mkdir -p $OUT
for e in ffma tc; do
  timeout 600 python bench.py --engine $e --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/c3_$e.log 2>&1
  timeout 600 python bench.py --engine $e --input dense --steps 10 --warmup 3 --no-cpu --no-e2e > $OUT/c3dense_$e.log 2>&1
done
