#!/bin/bash
# GPU-box check used during development: gpu tests + one bench line per config.
# usage: bash scripts/gpu_check.sh [configs...]
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1
  echo "tests rc=$?" >> gpurun_out/gputests.log
  tail -3 gpurun_out/gputests.log
fi
CFGS=${@:-C5 C4 C3a C3b C2a C2b C1}
for c in $CFGS; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 $BENCH_ARGS > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c rc=$?"
done
