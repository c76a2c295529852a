#!/bin/bash
# usage: bash scripts/ncu_top.sh <name> <kernel regex> <skip> <bench args...>
# full ncu capture of one launch of the matching kernel (after a plain run exits 0)
mkdir -p gpurun_out
name=$1; kre=$2; skip=$3; shift 3
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/ncu_${name}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c ${COUNT:-1} \
    -o gpurun_out/prof_${name} -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu "$@" > gpurun_out/ncu_${name}.log 2>&1
echo "ncu rc=$?"
