#!/bin/bash
# usage: bash scripts/ncu_k.sh <name> <kernel regex> <skip> <bench args...>   (no plain pre-run)
mkdir -p gpurun_out
name=$1; kre=$2; skip=$3; shift 3
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c 1 \
    -o gpurun_out/prof_${name} -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/ncu_${name}.log 2>&1
echo "ncu rc=$?"
