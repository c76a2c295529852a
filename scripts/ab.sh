#!/bin/bash
# A/B helper: bash scripts/ab.sh "ENV=1 ENV2=x" config...   (bench lines -> gpurun_out/ab_<tag>_<cfg>.json)
mkdir -p gpurun_out
tag=$1; envs=$2; shift 2
for c in "$@"; do
  env $envs timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/ab_${tag}_$c.json 2> gpurun_out/ab_${tag}_$c.err
  echo "$tag $c rc=$?"
done
