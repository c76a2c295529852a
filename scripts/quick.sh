#!/bin/bash
# quick GPU check: tests, then C5 and C4 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/q_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/q_tests.log
for c in ${@:-C5 C4}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/q_bench_$c.json 2> gpurun_out/q_bench_$c.err
  echo "bench $c rc=$?"; tail -2 gpurun_out/q_bench_$c.err
done
