#!/bin/bash
# one full ncu capture of kernels matching $1 in a C5-style bench run (after a plain run)
# usage: bash scripts/prof_k.sh <tag> <regex> <skip> <count> [bench args...]
tag=$1; kre=$2; skip=$3; cnt=$4; shift 4
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph "$@" > gpurun_out/${tag}_plain.json 2> gpurun_out/${tag}_plain.err && \
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c $cnt \
    -o gpurun_out/${tag} -f python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu --no-graph "$@" > gpurun_out/${tag}_ncu.log 2>&1
echo "prof rc=$?"
