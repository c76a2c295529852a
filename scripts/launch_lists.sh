#!/bin/bash
# ncu launch lists (duration + DRAM bytes per kernel) of the smaller BASELINE configs,
# each after the same command has exited 0 without ncu.  Outputs gpurun_out/ll_<cfg>.csv
mkdir -p gpurun_out
for c in "$@"; do
  python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu > gpurun_out/ll_plain_$c.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file gpurun_out/ll_$c.csv python bench.py --config $c --steps 2 --warmup 1 --no-e2e --no-cpu \
      > gpurun_out/ll_ncu_$c.log 2>&1
  echo "$c rc=$?"
done
